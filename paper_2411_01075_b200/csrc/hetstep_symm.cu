// Fused uneven collectives over NVLink 5 / NVSwitch on a symmetric buffer
// (same byte offset on every rank; peer-mapped and, when the fabric supports
// it, bound to an NVLS multicast object).
//
//   het_symm_allgather_pack  — rank r reads its fp32 master range, rounds to
//     bf16 and stores it ONCE through the multicast address: the switch
//     replicates it into every rank's gathered unit (owner egress = s_r, not
//     (N-1) s_r). Fuses kernel (1) "pack" with collective (2).
//   het_symm_reduce_scatter  — rank r reads its own range of the unit
//     accumulator with multimem.ld_reduce: the switch sums the N ranks' (Eq. 1
//     pre-scaled) fp32 accumulators in flight and returns one stream, which
//     is written straight into r's fp32 grad shard. Collective (3) as a
//     single kernel, no staging.
//   Without multicast both fall back to peer-pointer stores/loads in the same
//   kernel (push AG, pull RS).
//
// Synchronisation is in-kernel: CTA b of every rank meets CTA b of every
// other rank on a per-(channel, kind, cta, src) signal slot carrying a
// monotonically increasing epoch (release/acquire at system scope). The
// start barrier orders "every rank finished producing / released the buffer"
// before the first remote access; the end barrier orders "all stores
// landed" (AG) or "all peers finished reading" (RS, optional). Spins are
// bounded: on timeout the kernel records HET_SYMM_TIMEOUT and exits instead of
// hanging the GPU.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>
#include <cstdlib>
#include <cstring>

#include "hetstep.h"
#include "hetstep_internal.cuh"

using het::fail;

namespace {

constexpr int kThreads = 512;
constexpr int kUnroll = 8;                   // independent 16-byte remote ops per thread
constexpr int kMaxCtas = HET_SYMM_MAX_CTAS;
// signal slot kinds: 0 start barrier, 1 end barrier, 2 pair-relay flag, 3 helper progress
constexpr int kKinds = 4;

// The CTA's index and count WITHIN ITS RANK's grid. A real launch runs one rank
// per grid (blockIdx.x, gridDim.x). The virtual-rank launch (het_symm_virtual)
// runs N ranks as ONE cooperative grid of N * ctas CTAs -- CTA b of rank r at
// blockIdx.x = r * ctas + b -- so all CTAs are co-resident by construction.
// Every barrier slot, grid-stride loop and "CTA 0" edge below uses these.
__shared__ int s_cta, s_ncta;

__device__ __forceinline__ void set_ctx(int cta, int ncta) {
  s_cta = cta;              // every thread writes the same value
  s_ncta = ncta;
  __syncthreads();
}
// Barrier spin limit (wall clock); het_tune(HET_TUNE_SYMM_TIMEOUT_MS) overrides it
// so a fault-injection test need not wait the full 10 s.
uint64_t g_spin_timeout_ns = 10ull * 1000 * 1000 * 1000;

__device__ int g_symm_status = 0;

// het_symm_status_async: the sticky status copied to `dst` (device memory or
// pinned host memory, which is device-mapped under UVA) stream-ordered after
// the step's collectives, so the host can check it without a device sync.
__global__ void status_copy_kernel(int32_t* dst) { *dst = *(volatile int*)&g_symm_status; }

struct Args {
  het_symm_t s;
  uint64_t data_off;       // byte offset of the unit (AG: bf16 unit, RS: fp32 acc)
  int64_t count;           // this rank's element count
  int64_t offset;          // this rank's element offset inside the unit
  uint32_t epoch;
  int channel;
  int end_barrier;
  // AG relay (HET_SYMM_RELAY, peer route only): my last relay_vecs body
  // vectors go to me and relay_to only, and relay_to forwards them; I forward
  // the last from_vecs body vectors of rank relay_from (count from_count at
  // from_offset). -1 / 0 = none.
  int relay_to = -1, relay_from = -1;
  int64_t relay_vecs = 0, from_count = 0, from_offset = 0, from_vecs = 0;
  uint64_t timeout_ns = 0;    // barrier spin limit (g_spin_timeout_ns at launch)
};

__device__ __forceinline__ uint32_t* slot(uint64_t owner_base, uint64_t signal_off, int channel,
                                          int kind, int cta, int src) {
  const uint64_t idx =
      ((static_cast<uint64_t>(channel) * kKinds + kind) * kMaxCtas + cta) * HET_MAX_RANKS + src;
  return reinterpret_cast<uint32_t*>(owner_base + signal_off + idx * 4);
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Copy the peer table from parameter space with compile-time indices (a
// dynamic index into a kernel parameter would force a local-memory copy).
#define HET_STAGE_PEERS(args, peer)                                   \
  do {                                                                \
    _Pragma("unroll") for (int i_ = 0; i_ < HET_MAX_RANKS; ++i_)       \
      if (threadIdx.x == i_) (peer)[i_] = (args).s.peer_base[i_];       \
  } while (0)

// CTA-pairwise cross-rank barrier (see file comment).
// Scalar view of het_symm_t held in registers (the peer table lives in smem).
struct Sym {
  int nranks, rank;
  uint64_t mc_base, signal_off, timeout_ns;
};

// Spin until the slot reaches `epoch`; on timeout record HET_SYMM_TIMEOUT
// (read back by het_symm_status / het_symm_status_async) and give up.
__device__ __forceinline__ void wait_epoch(const uint32_t* p, uint32_t epoch, uint64_t timeout_ns) {
  const uint64_t t0 = globaltimer_ns();
  while (static_cast<int32_t>(ld_acquire_sys(p) - epoch) < 0) {
    if (globaltimer_ns() - t0 > timeout_ns) {
      atomicExch(&g_symm_status, HET_SYMM_TIMEOUT);
      break;
    }
  }
}

// Device-resident barrier epochs (CUDA-graph replay of a multi-rank step): the
// rank's base epoch per channel lives in its own signal area, right after the
// barrier slots. A launch whose epoch has HET_SYMM_EPOCH_DEVICE set runs at
// base[channel] + (epoch & ~HET_SYMM_EPOCH_DEVICE); het_symm_epoch_add advances
// the base, stream-ordered after the channel's last launch of the step, so the
// same captured arguments yield fresh epochs on every replay.
__host__ __device__ constexpr uint64_t slot_bytes() {
  return static_cast<uint64_t>(HET_SYMM_CHANNELS) * kKinds * kMaxCtas * HET_MAX_RANKS * 4;
}

__device__ __forceinline__ uint32_t* epoch_base(uint64_t own_base, uint64_t signal_off,
                                                int channel) {
  return reinterpret_cast<uint32_t*>(own_base + signal_off + slot_bytes()) + channel;
}

// Every thread of the CTA returns the same value (the base is only written by
// het_symm_epoch_add / _set, stream-ordered against the collectives).
__device__ __forceinline__ uint32_t launch_epoch(const Args& a, const uint64_t* peer) {
  __syncthreads();                                  // peer table staged
  if (!(a.epoch & HET_SYMM_EPOCH_DEVICE)) return a.epoch;
  const volatile uint32_t* b = epoch_base(peer[a.s.rank], a.s.signal_off, a.channel);
  return *b + (a.epoch & ~HET_SYMM_EPOCH_DEVICE);
}

__global__ void epoch_update_kernel(uint32_t* base, uint32_t v, int add) {
  *base = add ? *base + v : v;
}

// `peer` is the CTA's shared copy of the peer base table.
__device__ void cross_barrier(const Sym& s, const uint64_t* peer, int channel, int kind,
                              uint32_t epoch) {
  __syncthreads();
  const int t = threadIdx.x;
  if (t < s.nranks) {
    __threadfence_system();
    st_release_sys(slot(peer[t], s.signal_off, channel, kind, s_cta, s.rank), epoch);
    wait_epoch(slot(peer[s.rank], s.signal_off, channel, kind, s_cta, t), epoch,
               s.timeout_ns);
  }
  __syncthreads();
}

__device__ __forceinline__ void mc_st_v4(uint64_t addr, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(addr),
               "f"(__uint_as_float(v.x)), "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)),
               "f"(__uint_as_float(v.w))
               : "memory");
}

__device__ __forceinline__ void mc_st_b32(uint64_t addr, uint32_t v) {
  asm volatile("multimem.st.relaxed.sys.global.bf16x2 [%0], %1;" ::"l"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ float4 mc_ldr_v4(uint64_t addr) {
  float4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(addr));
  return r;
}

__device__ __forceinline__ float mc_ldr_f32(uint64_t addr) {
  float r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];"
               : "=f"(r)
               : "l"(addr)
               : "memory");
  return r;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// ---------------------------------------------------------------- all-gather

// Element geometry of one rank's bf16 range at byte offset dst0: [0,h1)
// 2-byte edge, [h1,h2) 4-byte words, nvec 16-byte vectors, then the tail.
// Host twin: ag_geometry() below (the relay plan must agree with it).
__host__ __device__ inline void ag_geometry(uint64_t dst0, int64_t n, int64_t* h1o, int64_t* h2o,
                                            int64_t* nveco) {
  int64_t h1 = (dst0 & 3) ? 1 : 0;
  if (h1 > n) h1 = n;
  int64_t h2 = h1 + static_cast<int64_t>(((16 - ((dst0 + h1 * 2) & 15)) & 15) / 2);
  if (h2 > n) h2 = n;
  *h1o = h1;
  *h2o = h2;
  *nveco = (n - h2) / 8;
}

// Pack body vectors [lo,hi) of my fp32 range and store each to the peers in
// `mask` (bit p = rank p); kUnroll vectors per thread in flight, all local
// loads issued before the remote stores.
template <int NR>
__device__ __forceinline__ void ag_push(const float* __restrict__ src, int64_t h2, int64_t lo,
                                        int64_t hi, uint64_t dst0, const uint64_t* peer, int nr,
                                        uint32_t mask, bool src_vec) {
  const int64_t gtid = static_cast<int64_t>(s_cta) * blockDim.x + threadIdx.x;
  const int64_t gsz = static_cast<int64_t>(s_ncta) * blockDim.x;
  for (int64_t v0 = lo + gtid; v0 < hi; v0 += gsz * kUnroll) {
    uint4 w[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t v = v0 + u * gsz;
      if (v < hi) {
        const float* p = src + h2 + v * 8;
        float f[8];
        if (src_vec) {
          const float4 x = __ldcs(reinterpret_cast<const float4*>(p));
          const float4 y = __ldcs(reinterpret_cast<const float4*>(p) + 1);
          f[0] = x.x; f[1] = x.y; f[2] = x.z; f[3] = x.w;
          f[4] = y.x; f[5] = y.y; f[6] = y.z; f[7] = y.w;
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = p[i];
        }
        w[u] = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]),
                          pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t v = v0 + u * gsz;
      if (v < hi) {
        const uint64_t off = dst0 + static_cast<uint64_t>(h2 + v * 8) * 2;
#pragma unroll
        for (int p = 0; p < (NR > 0 ? NR : HET_MAX_RANKS); ++p)
          if (p < nr && ((mask >> p) & 1u)) *reinterpret_cast<uint4*>(peer[p] + off) = w[u];
      }
    }
  }
}

// Forward body vectors [lo,hi) of another rank's range (already landed in my
// copy of the unit) to the peers in `mask`. Same vector -> CTA mapping as
// ag_push, so CTA b forwards exactly what the owner's CTA b sent it.
template <int NR>
__device__ __forceinline__ void ag_forward(int64_t h2, int64_t lo, int64_t hi, uint64_t dst0,
                                           const uint64_t* peer, int me, int nr, uint32_t mask) {
  const int64_t gtid = static_cast<int64_t>(s_cta) * blockDim.x + threadIdx.x;
  const int64_t gsz = static_cast<int64_t>(s_ncta) * blockDim.x;
  for (int64_t v0 = lo + gtid; v0 < hi; v0 += gsz * kUnroll) {
    uint4 w[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t v = v0 + u * gsz;
      if (v < hi)
        w[u] = __ldcg(reinterpret_cast<const uint4*>(peer[me] + dst0 +
                                                     static_cast<uint64_t>(h2 + v * 8) * 2));
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t v = v0 + u * gsz;
      if (v < hi) {
        const uint64_t off = dst0 + static_cast<uint64_t>(h2 + v * 8) * 2;
#pragma unroll
        for (int p = 0; p < (NR > 0 ? NR : HET_MAX_RANKS); ++p)
          if (p < nr && ((mask >> p) & 1u)) *reinterpret_cast<uint4*>(peer[p] + off) = w[u];
      }
    }
  }
}

template <bool MC, int NR>
__device__ __forceinline__ void symm_ag_kernel_body(const float* __restrict__ src,
                                                           const Args& a) {
  __shared__ uint64_t peer[HET_MAX_RANKS];
  HET_STAGE_PEERS(a, peer);
  const Sym s{a.s.nranks, a.s.rank, a.s.mc_base, a.s.signal_off, a.timeout_ns};
  const uint32_t ep = launch_epoch(a, peer);
  cross_barrier(s, peer, a.channel, 0, ep);   // every rank released its copy of the unit
  const int64_t n = a.count;
  const uint64_t dst0 = a.data_off + static_cast<uint64_t>(a.offset) * 2;  // byte offset
  const int nr = NR > 0 ? NR : s.nranks;   // compile-time for 2/4/8 ranks: loops unroll
  // element ranges: [0,h1) 2-byte edge, [h1,h2) 4-byte words, body 16-byte vectors, tail
  int64_t h1 = (dst0 & 3) ? 1 : 0;
  if (h1 > n) h1 = n;
  int64_t h2 = h1 + static_cast<int64_t>(((16 - ((dst0 + h1 * 2) & 15)) & 15) / 2);
  if (h2 > n) h2 = n;
  const int64_t nvec = (n - h2) / 8;
  const int64_t body_end = h2 + nvec * 8;
  const int64_t gtid = static_cast<int64_t>(s_cta) * blockDim.x + threadIdx.x;
  const int64_t gsz = static_cast<int64_t>(s_ncta) * blockDim.x;
  // body: 8 bf16 per 16-byte multicast store; kUnroll vectors per thread in
  // flight (all local loads issued before the remote stores)
  const bool src_vec = ((reinterpret_cast<uintptr_t>(src + h2)) & 15) == 0;
  if (!MC && (a.relay_to >= 0 || a.relay_from >= 0)) {
    // relay route: the relayed tail first (to me + my relay), flag it, then
    // the direct body; the relay forwards after its own body so its egress
    // carries part of the big owner's.
    const uint32_t all = (nr >= 32) ? 0xffffffffu : ((1u << nr) - 1u);
    int64_t direct = nvec;
    if (a.relay_to >= 0) {
      direct = nvec - a.relay_vecs;
      ag_push<NR>(src, h2, direct, nvec, dst0, peer, nr,
                  (1u << s.rank) | (1u << a.relay_to), src_vec);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence_system();
        st_release_sys(slot(peer[a.relay_to], s.signal_off, a.channel, 2, s_cta, s.rank),
                       ep);
      }
    }
    ag_push<NR>(src, h2, 0, direct, dst0, peer, nr, all, src_vec);
    if (a.relay_from >= 0) {
      if (threadIdx.x == 0) {
        wait_epoch(slot(peer[s.rank], s.signal_off, a.channel, 2, s_cta, a.relay_from),
                   ep, s.timeout_ns);
      }
      __syncthreads();
      const uint64_t fdst0 = a.data_off + static_cast<uint64_t>(a.from_offset) * 2;
      int64_t fh1, fh2, fnvec;
      ag_geometry(fdst0, a.from_count, &fh1, &fh2, &fnvec);
      ag_forward<NR>(fh2, fnvec - a.from_vecs, fnvec, fdst0, peer, s.rank, nr,
                     all & ~((1u << s.rank) | (1u << a.relay_from)));
    }
  } else
  for (int64_t v0 = gtid; v0 < nvec; v0 += gsz * kUnroll) {
    uint4 w[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t v = v0 + u * gsz;
      if (v < nvec) {
        const float* p = src + h2 + v * 8;
        float f[8];
        if (src_vec) {
          const float4 x = __ldcs(reinterpret_cast<const float4*>(p));
          const float4 y = __ldcs(reinterpret_cast<const float4*>(p) + 1);
          f[0] = x.x; f[1] = x.y; f[2] = x.z; f[3] = x.w;
          f[4] = y.x; f[5] = y.y; f[6] = y.z; f[7] = y.w;
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = p[i];
        }
        w[u] = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]),
                          pack_bf16x2(f[4], f[5]), pack_bf16x2(f[6], f[7]));
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t v = v0 + u * gsz;
      if (v < nvec) {
        const uint64_t off = dst0 + static_cast<uint64_t>(h2 + v * 8) * 2;
        if (MC) {
          mc_st_v4(s.mc_base + off, w[u]);
        } else {
#pragma unroll
          for (int p = 0; p < nr; ++p) *reinterpret_cast<uint4*>(peer[p] + off) = w[u];
        }
      }
    }
  }
  // edges (CTA 0): 4-byte pairs via multicast, a lone 2-byte element via peer stores
  if (s_cta == 0) {
    auto pair = [&](int64_t e) {
      const uint64_t off = dst0 + static_cast<uint64_t>(e) * 2;
      const uint32_t w = pack_bf16x2(src[e], src[e + 1]);
      if (MC)
        mc_st_b32(s.mc_base + off, w);
      else
        for (int p = 0; p < nr; ++p) *reinterpret_cast<uint32_t*>(peer[p] + off) = w;
    };
    auto single = [&](int64_t e) {
      const uint64_t off = dst0 + static_cast<uint64_t>(e) * 2;
      const __nv_bfloat16 h = __float2bfloat16_rn(src[e]);
      for (int p = 0; p < nr; ++p) *reinterpret_cast<__nv_bfloat16*>(peer[p] + off) = h;
    };
    const int t = threadIdx.x;
    if (t == 0 && h1 == 1) single(0);
    for (int64_t e = h1 + 2 * t; e + 1 < h2; e += 2 * blockDim.x) pair(e);
    if (t == 0 && (h2 - h1) % 2 == 1) single(h2 - 1);
    // tail after the body: pairs from an even (4-byte aligned) start, then a lone element
    for (int64_t e = body_end + 2 * t; e + 1 < n; e += 2 * blockDim.x) pair(e);
    if (t == 0 && (n - body_end) % 2 == 1) single(n - 1);
  }
  cross_barrier(s, peer, a.channel, 1, ep);   // every rank's stores have landed
}

template <bool MC, int NR>
__global__ void __launch_bounds__(kThreads) symm_ag_kernel(const float* __restrict__ src,
                                                           const __grid_constant__ Args a) {
  set_ctx(blockIdx.x, gridDim.x);
  symm_ag_kernel_body<MC, NR>(src, a);
}

// ---------------------------------------------------------------- reduce-scatter

__device__ __forceinline__ void store4(float* out, int64_t e, const float4& r, bool vec) {
  if (vec) {
    __stcs(reinterpret_cast<float4*>(out + e), r);
  } else {
    out[e] = r.x;
    out[e + 1] = r.y;
    out[e + 2] = r.z;
    out[e + 3] = r.w;
  }
}

template <bool MC, int NR>
__device__ __forceinline__ void symm_rs_kernel_body(float* __restrict__ out, const Args& a) {
  __shared__ uint64_t peer[HET_MAX_RANKS];
  HET_STAGE_PEERS(a, peer);
  const Sym s{a.s.nranks, a.s.rank, a.s.mc_base, a.s.signal_off, a.timeout_ns};
  const uint32_t ep = launch_epoch(a, peer);
  cross_barrier(s, peer, a.channel, 0, ep);   // every rank's accumulator is final
  const int64_t n = a.count;
  const uint64_t src0 = a.data_off + static_cast<uint64_t>(a.offset) * 4;
  const int nr = NR > 0 ? NR : s.nranks;   // compile-time for 2/4/8 ranks: loops unroll
  int64_t head = static_cast<int64_t>(((16 - (src0 & 15)) & 15) / 4);
  if (head > n) head = n;
  const int64_t nvec = (n - head) / 4;
  const int64_t body_end = head + nvec * 4;
  const bool out_vec = ((reinterpret_cast<uintptr_t>(out + head)) & 15) == 0;
  const int64_t gtid = static_cast<int64_t>(s_cta) * blockDim.x + threadIdx.x;
  const int64_t gsz = static_cast<int64_t>(s_ncta) * blockDim.x;
  if (MC) {
    for (int64_t v0 = gtid; v0 < nvec; v0 += gsz * kUnroll) {
      float4 r[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {        // kUnroll switch reductions in flight
        const int64_t v = v0 + u * gsz;
        if (v < nvec) r[u] = mc_ldr_v4(s.mc_base + src0 + static_cast<uint64_t>(head + v * 4) * 4);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t v = v0 + u * gsz;
        if (v < nvec) store4(out, head + v * 4, r[u], out_vec);
      }
    }
  } else {
    // peer pull: all (vector, rank) loads of a batch issued before any add
    constexpr int kB = NR > 0 ? (16 / NR > 1 ? 16 / NR : 2) : 2;
    for (int64_t v0 = gtid; v0 < nvec; v0 += gsz * kB) {
      float4 x[kB][NR > 0 ? NR : HET_MAX_RANKS];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int64_t v = v0 + u * gsz;
        if (v < nvec) {
          const uint64_t off = src0 + static_cast<uint64_t>(head + v * 4) * 4;
#pragma unroll
          for (int p = 0; p < (NR > 0 ? NR : HET_MAX_RANKS); ++p)
            if (p < nr) x[u][p] = __ldcg(reinterpret_cast<const float4*>(peer[p] + off));
        }
      }
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        const int64_t v = v0 + u * gsz;
        if (v < nvec) {
          float4 r = x[u][0];
#pragma unroll
          for (int p = 1; p < (NR > 0 ? NR : HET_MAX_RANKS); ++p) {
            if (p < nr) {
              r.x += x[u][p].x;
              r.y += x[u][p].y;
              r.z += x[u][p].z;
              r.w += x[u][p].w;
            }
          }
          store4(out, head + v * 4, r, out_vec);
        }
      }
    }
  }
  if (s_cta == 0) {
    auto one = [&](int64_t e) {
      const uint64_t off = src0 + static_cast<uint64_t>(e) * 4;
      float r = 0.f;
      if (MC) {
        r = mc_ldr_f32(s.mc_base + off);
      } else {
        for (int p = 0; p < nr; ++p) r += *reinterpret_cast<const float*>(peer[p] + off);
      }
      out[e] = r;
    };
    for (int64_t e = threadIdx.x; e < head; e += blockDim.x) one(e);
    for (int64_t e = body_end + threadIdx.x; e < n; e += blockDim.x) one(e);
  }
  if (a.end_barrier) cross_barrier(s, peer, a.channel, 1, ep);  // peers done reading my acc
}

template <bool MC, int NR>
__global__ void __launch_bounds__(kThreads) symm_rs_kernel(float* __restrict__ out, const __grid_constant__ Args a) {
  set_ctx(blockIdx.x, gridDim.x);
  symm_rs_kernel_body<MC, NR>(out, a);
}

// ---------------------------------------------------------------- reduce-scatter, bf16 wire

struct Weights {
  float w[HET_MAX_RANKS];
};

__device__ __forceinline__ void bf8_to_f(const uint4& raw, float (&f)[8]) {
  const uint32_t u[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float((u[i] & 0xffffu) << 16);
    f[2 * i + 1] = __uint_as_float(u[i] & 0xffff0000u);
  }
}

template <int NR>
__device__ __forceinline__ void symm_rs_bf16_kernel_body(float* __restrict__ out,
                                                                const Args& a,
                                                                const Weights& wt) {
  __shared__ uint64_t peer[HET_MAX_RANKS];
  HET_STAGE_PEERS(a, peer);
  const Sym s{a.s.nranks, a.s.rank, a.s.mc_base, a.s.signal_off, a.timeout_ns};
  const uint32_t ep = launch_epoch(a, peer);
  cross_barrier(s, peer, a.channel, 0, ep);   // every rank's gradient is staged
  const int64_t n = a.count;
  const uint64_t src0 = a.data_off + static_cast<uint64_t>(a.offset) * 2;
  const int nr = NR > 0 ? NR : s.nranks;
  constexpr int kMaxR = NR > 0 ? NR : HET_MAX_RANKS;
  int64_t head = static_cast<int64_t>(((16 - (src0 & 15)) & 15) / 2);
  if (head > n) head = n;
  const int64_t nvec = (n - head) / 8;
  const int64_t body_end = head + nvec * 8;
  const bool out_vec = ((reinterpret_cast<uintptr_t>(out + head)) & 15) == 0;
  const int64_t gtid = static_cast<int64_t>(s_cta) * blockDim.x + threadIdx.x;
  const int64_t gsz = static_cast<int64_t>(s_ncta) * blockDim.x;
  constexpr int kB = NR > 0 ? (16 / NR > 1 ? 16 / NR : 2) : 2;   // vectors per batch
  for (int64_t v0 = gtid; v0 < nvec; v0 += gsz * kB) {
    uint4 x[kB][kMaxR];
#pragma unroll
    for (int u = 0; u < kB; ++u) {          // all (vector, rank) loads before any math
      const int64_t v = v0 + u * gsz;
      if (v < nvec) {
        const uint64_t off = src0 + static_cast<uint64_t>(head + v * 8) * 2;
#pragma unroll
        for (int p = 0; p < kMaxR; ++p)      // ranks with no batch (w = 0) are not read
          if (p < nr && wt.w[p] != 0.f)
            x[u][p] = __ldcg(reinterpret_cast<const uint4*>(peer[p] + off));
      }
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int64_t v = v0 + u * gsz;
      if (v < nvec) {
        // explicit rounding: fl(w_j g_j) summed in rank order, exactly as the fp32
        // route's (accumulate FIRST, then peer-pull sum) arithmetic
        float r[8], f[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = 0.f;
#pragma unroll
        for (int p = 0; p < kMaxR; ++p) {
          if (p < nr && wt.w[p] != 0.f) {
            bf8_to_f(x[u][p], f);
#pragma unroll
            for (int i = 0; i < 8; ++i) r[i] = __fadd_rn(r[i], __fmul_rn(wt.w[p], f[i]));
          }
        }
        const int64_t e = head + v * 8;
        if (out_vec) {
          __stcs(reinterpret_cast<float4*>(out + e), make_float4(r[0], r[1], r[2], r[3]));
          __stcs(reinterpret_cast<float4*>(out + e + 4), make_float4(r[4], r[5], r[6], r[7]));
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) out[e + i] = r[i];
        }
      }
    }
  }
  if (s_cta == 0) {
    auto one = [&](int64_t e) {
      const uint64_t off = src0 + static_cast<uint64_t>(e) * 2;
      float r = 0.f;
      for (int p = 0; p < nr; ++p) {
        if (wt.w[p] == 0.f) continue;
        const float g = __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(peer[p] + off));
        r = __fadd_rn(r, __fmul_rn(wt.w[p], g));
      }
      out[e] = r;
    };
    for (int64_t e = threadIdx.x; e < head; e += blockDim.x) one(e);
    for (int64_t e = body_end + threadIdx.x; e < n; e += blockDim.x) one(e);
  }
  if (a.end_barrier) cross_barrier(s, peer, a.channel, 1, ep);  // peers done reading mine
}

template <int NR>
__global__ void __launch_bounds__(kThreads) symm_rs_bf16_kernel(float* __restrict__ out,
                                                                const __grid_constant__ Args a,
                                                                const __grid_constant__ Weights wt) {
  set_ctx(blockIdx.x, gridDim.x);
  symm_rs_bf16_kernel_body<NR>(out, a, wt);
}


// ---------------------------------------------------------------- helper relay
//
// HET_SYMM_HELPERS: a heavy owner hands pieces of its range to light ranks
// ("helpers"), which finish the collective for those pieces:
//   all-gather:      the owner pushes a piece to its helper only; the helper
//                    forwards it to the other N-2 ranks.
//   reduce-scatter:  the helper reduces the piece over all N ranks (pull) into
//                    a staging copy in its own buffer; the owner pulls the
//                    reduced piece instead of N-1 raw ones.
// A single owner at N ranks thus moves S bytes over its link instead of
// (N-1) S (plain push / pull) and every helper link carries about S as well
// (helper_plan). Pieces are ranges of the owner's body vectors and are
// streamed in grid-stride iterations; after iteration k of a piece the
// producing CTA b release-stores a progress count into slot (kind 3, cta b)
// of the consumer, whose CTA b acquires it before consuming iteration k: the
// same vector -> CTA mapping on both sides, so only CTA b's own progress is
// awaited (a pipelined, CTA-pairwise handoff).

struct HArgs {
  int64_t direct;                        // my body vectors [0, direct) go the plain way
  int n_own, n_help;
  int own_peer[HET_MAX_RANKS];           // my pieces: helper rank, body vector range
  int64_t own_lo[HET_MAX_RANKS], own_hi[HET_MAX_RANKS];
  int help_peer[HET_MAX_RANKS];          // pieces I help with: owner rank, range,
  int64_t help_lo[HET_MAX_RANKS], help_hi[HET_MAX_RANKS];   // owner's count / offset
  int64_t help_count[HET_MAX_RANKS], help_offset[HET_MAX_RANKS];
  int gran;                              // iterations per progress signal
  uint64_t stage_off;                    // RS: fp32 staging region (in place for fp32)
};

__device__ __forceinline__ int64_t iters_of(int64_t lo, int64_t hi, int64_t per_iter) {
  return hi > lo ? (hi - lo + per_iter - 1) / per_iter : 0;
}

// progress value after iteration k (signalled when (k+1) % gran == 0 or k is last)
__device__ __forceinline__ uint32_t progress(uint32_t epoch, int64_t k, int gran) {
  return epoch * 4096u + static_cast<uint32_t>(k / gran + 1);
}

__device__ __forceinline__ void signal_progress(uint64_t owner_base, const Sym& s, int channel,
                                                uint32_t v) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    st_release_sys(slot(owner_base, s.signal_off, channel, 3, s_cta, s.rank), v);
  }
}

__device__ __forceinline__ void await_progress(const uint64_t* peer, const Sym& s, int channel,
                                               int src, uint32_t v) {
  if (threadIdx.x == 0)
    wait_epoch(slot(peer[s.rank], s.signal_off, channel, 3, s_cta, src), v, s.timeout_ns);
  __syncthreads();
}

template <int NR>
__device__ __forceinline__ void symm_ag_help_kernel_body(const float* __restrict__ src,
                                                                const Args& a,
                                                                const HArgs& h) {
  __shared__ uint64_t peer[HET_MAX_RANKS];
  HET_STAGE_PEERS(a, peer);
  const Sym s{a.s.nranks, a.s.rank, a.s.mc_base, a.s.signal_off, a.timeout_ns};
  const uint32_t ep = launch_epoch(a, peer);
  cross_barrier(s, peer, a.channel, 0, ep);   // every rank released its copy of the unit
  const int nr = NR > 0 ? NR : s.nranks;
  const uint32_t all = (nr >= 32) ? 0xffffffffu : ((1u << nr) - 1u);
  const int me = s.rank;
  const int64_t n = a.count;
  const uint64_t dst0 = a.data_off + static_cast<uint64_t>(a.offset) * 2;
  int64_t h1, h2, nvec;
  ag_geometry(dst0, n, &h1, &h2, &nvec);
  const bool src_vec = ((reinterpret_cast<uintptr_t>(src + h2)) & 15) == 0;
  const int64_t per_iter = static_cast<int64_t>(s_ncta) * blockDim.x * kUnroll;
  // 1) my pieces to their helpers only (interleaved, so every helper starts early)
  int64_t kmax = 0;
  for (int p = 0; p < h.n_own; ++p) {
    const int64_t k = iters_of(h.own_lo[p], h.own_hi[p], per_iter);
    kmax = k > kmax ? k : kmax;
  }
  for (int64_t k = 0; k < kmax; ++k) {
    for (int p = 0; p < h.n_own; ++p) {
      const int64_t kp = iters_of(h.own_lo[p], h.own_hi[p], per_iter);
      if (k >= kp) continue;
      const int64_t lo = h.own_lo[p] + k * per_iter;
      const int64_t hi = lo + per_iter < h.own_hi[p] ? lo + per_iter : h.own_hi[p];
      ag_push<NR>(src, h2, lo, hi, dst0, peer, nr, (1u << me) | (1u << h.own_peer[p]), src_vec);
      if ((k + 1) % h.gran == 0 || k + 1 == kp)
        signal_progress(peer[h.own_peer[p]], s, a.channel, progress(ep, k, h.gran));
    }
  }
  // 2) my direct body vectors to every rank
  ag_push<NR>(src, h2, 0, h.direct, dst0, peer, nr, all, src_vec);
  // 3) forward the pieces I help with (they landed in my copy of the unit)
  kmax = 0;
  for (int q = 0; q < h.n_help; ++q) {
    const int64_t k = iters_of(h.help_lo[q], h.help_hi[q], per_iter);
    kmax = k > kmax ? k : kmax;
  }
  for (int64_t k = 0; k < kmax; ++k) {
    for (int q = 0; q < h.n_help; ++q) {
      const int64_t kq = iters_of(h.help_lo[q], h.help_hi[q], per_iter);
      if (k >= kq) continue;
      const int owner = h.help_peer[q];
      await_progress(peer, s, a.channel, owner, progress(ep, k, h.gran));
      const uint64_t fdst0 = a.data_off + static_cast<uint64_t>(h.help_offset[q]) * 2;
      int64_t fh1, fh2, fnvec;
      ag_geometry(fdst0, h.help_count[q], &fh1, &fh2, &fnvec);
      const int64_t lo = h.help_lo[q] + k * per_iter;
      const int64_t hi = lo + per_iter < h.help_hi[q] ? lo + per_iter : h.help_hi[q];
      ag_forward<NR>(fh2, lo, hi, fdst0, peer, me, nr, all & ~((1u << me) | (1u << owner)));
    }
  }
  // 4) edges of my range (CTA 0), straight to every rank
  if (s_cta == 0) {
    const int64_t body_end = h2 + nvec * 8;
    auto pair = [&](int64_t e) {
      const uint32_t w = pack_bf16x2(src[e], src[e + 1]);
      for (int p = 0; p < nr; ++p)
        *reinterpret_cast<uint32_t*>(peer[p] + dst0 + static_cast<uint64_t>(e) * 2) = w;
    };
    auto single = [&](int64_t e) {
      const __nv_bfloat16 v = __float2bfloat16_rn(src[e]);
      for (int p = 0; p < nr; ++p)
        *reinterpret_cast<__nv_bfloat16*>(peer[p] + dst0 + static_cast<uint64_t>(e) * 2) = v;
    };
    const int t = threadIdx.x;
    if (t == 0 && h1 == 1) single(0);
    for (int64_t e = h1 + 2 * t; e + 1 < h2; e += 2 * blockDim.x) pair(e);
    if (t == 0 && (h2 - h1) % 2 == 1) single(h2 - 1);
    for (int64_t e = body_end + 2 * t; e + 1 < n; e += 2 * blockDim.x) pair(e);
    if (t == 0 && (n - body_end) % 2 == 1) single(n - 1);
  }
  cross_barrier(s, peer, a.channel, 1, ep);   // every rank's stores have landed
}

template <int NR>
__global__ void __launch_bounds__(kThreads) symm_ag_help_kernel(const float* __restrict__ src,
                                                                const __grid_constant__ Args a,
                                                                const __grid_constant__ HArgs h) {
  set_ctx(blockIdx.x, gridDim.x);
  symm_ag_help_kernel_body<NR>(src, a, h);
}

// Reduce-scatter element geometry of a rank's range: 16-byte vectors of VE
// elements (4 fp32 or 8 bf16) after a head of unaligned elements.
template <bool BF16>
__device__ __forceinline__ void rs_geometry(uint64_t data_off, int64_t offset, int64_t n,
                                            int64_t* head, int64_t* nvec) {
  constexpr int ES = BF16 ? 2 : 4, VE = 16 / ES;
  const uint64_t src0 = data_off + static_cast<uint64_t>(offset) * ES;
  int64_t hd = static_cast<int64_t>(((16 - (src0 & 15)) & 15) / ES);
  if (hd > n) hd = n;
  *head = hd;
  *nvec = (n - hd) / VE;
}

// One vector (VE elements at element e of the unit) reduced over all ranks in
// rank order with explicit rounding: fp32 sum, or sum of fl(w_j * g_j).
template <int NR, bool BF16>
struct RsVec {
  static constexpr int VE = BF16 ? 8 : 4;
  static constexpr int kMaxR = NR > 0 ? NR : HET_MAX_RANKS;
  float r[VE];
  uint4 x[kMaxR];
  // issue the N peer loads of one vector (the caller batches several vectors'
  // loads before any combine, for memory-level parallelism)
  __device__ __forceinline__ void load(const uint64_t* peer, int nr, uint64_t byte_off,
                                       const Weights& wt) {
#pragma unroll
    for (int p = 0; p < kMaxR; ++p)
      if (p < nr && (!BF16 || wt.w[p] != 0.f))
        x[p] = __ldcg(reinterpret_cast<const uint4*>(peer[p] + byte_off));
  }
  __device__ __forceinline__ void reduce(const uint64_t* peer, int nr, uint64_t byte_off,
                                         const Weights& wt) {
    load(peer, nr, byte_off, wt);
    combine(nr, wt);
  }
  __device__ __forceinline__ void combine(int nr, const Weights& wt) {
#pragma unroll
    for (int i = 0; i < VE; ++i) r[i] = 0.f;
    bool first = true;
#pragma unroll
    for (int p = 0; p < kMaxR; ++p) {
      if (p >= nr) continue;
      if (BF16) {
        if (wt.w[p] == 0.f) continue;
        float f[8];
        bf8_to_f(x[p], f);
#pragma unroll
        for (int i = 0; i < VE; ++i) r[i] = __fadd_rn(r[i], __fmul_rn(wt.w[p], f[i]));
      } else {
        const float f[4] = {__uint_as_float(x[p].x), __uint_as_float(x[p].y),
                            __uint_as_float(x[p].z), __uint_as_float(x[p].w)};
#pragma unroll
        for (int i = 0; i < VE; ++i) r[i] = first ? f[i] : __fadd_rn(r[i], f[i]);
        first = false;
      }
    }
  }
};

// MC (fp32 only, HET_SYMM_HELPERS_MC): the helpers and the owner's direct part
// reduce through the switch (multimem.ld_reduce: one stream of sums in, 4 B per
// element) instead of pulling N-1 peers' ranges; the owner still pulls the
// staged sums. Not rank-ordered: within 1e-5 of the fp64 oracle, like the
// multicast route.
template <int NR, bool BF16, bool MC = false>
__device__ __forceinline__ void symm_rs_help_kernel_body(float* __restrict__ out,
                                                                const Args& a,
                                                                const HArgs& h,
                                                                const Weights& wt) {
  __shared__ uint64_t peer[HET_MAX_RANKS];
  HET_STAGE_PEERS(a, peer);
  const Sym s{a.s.nranks, a.s.rank, a.s.mc_base, a.s.signal_off, a.timeout_ns};
  const uint32_t ep = launch_epoch(a, peer);
  cross_barrier(s, peer, a.channel, 0, ep);   // every rank's input is final
  const int nr = NR > 0 ? NR : s.nranks;
  constexpr int ES = BF16 ? 2 : 4, VE = 16 / ES;
  const int64_t gtid = static_cast<int64_t>(s_cta) * blockDim.x + threadIdx.x;
  const int64_t gsz = static_cast<int64_t>(s_ncta) * blockDim.x;
  const int64_t per_iter = gsz * kUnroll;
  // 1) helper: reduce the owners' pieces into my staging copy, signal each iteration
  int64_t kmax = 0;
  for (int q = 0; q < h.n_help; ++q) {
    const int64_t k = iters_of(h.help_lo[q], h.help_hi[q], per_iter);
    kmax = k > kmax ? k : kmax;
  }
  for (int64_t k = 0; k < kmax; ++k) {
    for (int q = 0; q < h.n_help; ++q) {
      const int64_t kq = iters_of(h.help_lo[q], h.help_hi[q], per_iter);
      if (k >= kq) continue;
      int64_t head, nv;
      rs_geometry<BF16>(a.data_off, h.help_offset[q], h.help_count[q], &head, &nv);
      const int64_t lo = h.help_lo[q] + k * per_iter;
      const int64_t hi = lo + per_iter < h.help_hi[q] ? lo + per_iter : h.help_hi[q];
      if (MC && !BF16) {           // the switch sums the N ranks' vectors
        constexpr int kM = 8;      // reduced vectors in flight per thread
        for (int64_t v0 = lo + gtid; v0 < hi; v0 += gsz * kM) {
          float4 r[kM];
#pragma unroll
          for (int u = 0; u < kM; ++u) {
            const int64_t v = v0 + u * gsz;
            if (v < hi)
              r[u] = mc_ldr_v4(s.mc_base + a.data_off +
                               static_cast<uint64_t>(h.help_offset[q] + head + v * VE) * ES);
          }
#pragma unroll
          for (int u = 0; u < kM; ++u) {
            const int64_t v = v0 + u * gsz;
            if (v < hi)
              __stcg(reinterpret_cast<float4*>(peer[s.rank] + h.stage_off + static_cast<uint64_t>(
                                                   h.help_offset[q] + head + v * VE) * 4), r[u]);
          }
        }
        if ((k + 1) % h.gran == 0 || k + 1 == kq)
          signal_progress(peer[h.help_peer[q]], s, a.channel, progress(ep, k, h.gran));
        continue;
      }
      // kB vectors' N loads in flight per thread before any combine
      constexpr int kB = NR > 0 ? (16 / NR > 2 ? 16 / NR : 2) : 2;
      for (int64_t v0 = lo + gtid; v0 < hi; v0 += gsz * kB) {
        RsVec<NR, BF16> rv[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int64_t v = v0 + u * gsz;
          if (v < hi)
            rv[u].load(peer, nr, a.data_off + static_cast<uint64_t>(
                                     h.help_offset[q] + head + v * VE) * ES, wt);
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int64_t v = v0 + u * gsz;
          if (v >= hi) continue;
          rv[u].combine(nr, wt);
          const int64_t e = h.help_offset[q] + head + v * VE;      // unit element
          float4* st = reinterpret_cast<float4*>(peer[s.rank] + h.stage_off +
                                                 static_cast<uint64_t>(e) * 4);
          __stcg(st, make_float4(rv[u].r[0], rv[u].r[1], rv[u].r[2], rv[u].r[3]));
          if (BF16)
            __stcg(st + 1, make_float4(rv[u].r[4 % VE], rv[u].r[5 % VE], rv[u].r[6 % VE],
                                       rv[u].r[7 % VE]));
        }
      }
      if ((k + 1) % h.gran == 0 || k + 1 == kq)
        signal_progress(peer[h.help_peer[q]], s, a.channel, progress(ep, k, h.gran));
    }
  }
  // 2) my direct vectors: reduce over all ranks straight into my shard
  const int64_t n = a.count;
  int64_t head, nvec;
  rs_geometry<BF16>(a.data_off, a.offset, n, &head, &nvec);
  const bool out_vec = ((reinterpret_cast<uintptr_t>(out + head)) & 15) == 0;
  auto put = [&](int64_t le, const float* r) {   // le: element of my range
    if (out_vec) {
      __stcs(reinterpret_cast<float4*>(out + le), make_float4(r[0], r[1], r[2], r[3]));
      if (BF16) __stcs(reinterpret_cast<float4*>(out + le + 4),
                       make_float4(r[4 % VE], r[5 % VE], r[6 % VE], r[7 % VE]));
    } else {
#pragma unroll
      for (int i = 0; i < VE; ++i) out[le + i] = r[i];
    }
  };
  for (int64_t v = gtid; v < h.direct; v += gsz) {
    const uint64_t off = a.data_off + static_cast<uint64_t>(a.offset + head + v * VE) * ES;
    if (MC && !BF16) {
      const float4 r4 = mc_ldr_v4(s.mc_base + off);
      const float r[4] = {r4.x, r4.y, r4.z, r4.w};
      put(head + v * VE, r);
      continue;
    }
    RsVec<NR, BF16> rv;
    rv.reduce(peer, nr, off, wt);
    put(head + v * VE, rv.r);
  }
  // 3) owner: pull my pieces, reduced by their helpers, as they become ready
  kmax = 0;
  for (int p = 0; p < h.n_own; ++p) {
    const int64_t k = iters_of(h.own_lo[p], h.own_hi[p], per_iter);
    kmax = k > kmax ? k : kmax;
  }
  for (int64_t k = 0; k < kmax; ++k) {
    for (int p = 0; p < h.n_own; ++p) {
      const int64_t kp = iters_of(h.own_lo[p], h.own_hi[p], per_iter);
      if (k >= kp) continue;
      await_progress(peer, s, a.channel, h.own_peer[p], progress(ep, k, h.gran));
      const uint64_t base = peer[h.own_peer[p]] + h.stage_off;
      const int64_t lo = h.own_lo[p] + k * per_iter;
      const int64_t hi = lo + per_iter < h.own_hi[p] ? lo + per_iter : h.own_hi[p];
      constexpr int kB = 4;                     // staged vectors in flight per thread
      for (int64_t v0 = lo + gtid; v0 < hi; v0 += gsz * kB) {
        float4 x[kB][VE / 4];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int64_t v = v0 + u * gsz;
          if (v < hi) {
            const float4* src4 = reinterpret_cast<const float4*>(
                base + static_cast<uint64_t>(a.offset + head + v * VE) * 4);
#pragma unroll
            for (int j = 0; j < VE / 4; ++j) x[u][j] = __ldcg(src4 + j);
          }
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int64_t v = v0 + u * gsz;
          if (v < hi) {
            float r[VE];
#pragma unroll
            for (int j = 0; j < VE / 4; ++j) {
              r[4 * j] = x[u][j].x; r[4 * j + 1] = x[u][j].y;
              r[4 * j + 2] = x[u][j].z; r[4 * j + 3] = x[u][j].w;
            }
            put(head + v * VE, r);
          }
        }
      }
    }
  }
  // 4) head / tail elements of my range (CTA 0), reduced directly
  if (s_cta == 0) {
    const int64_t body_end = head + nvec * VE;
    auto one = [&](int64_t le) {
      const uint64_t off = a.data_off + static_cast<uint64_t>(a.offset + le) * ES;
      float r = 0.f;
      bool first = true;
      for (int p = 0; p < nr; ++p) {
        if (BF16) {
          if (wt.w[p] == 0.f) continue;
          const float g = __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(peer[p] + off));
          r = __fadd_rn(r, __fmul_rn(wt.w[p], g));
        } else {
          const float g = *reinterpret_cast<const float*>(peer[p] + off);
          r = first ? g : __fadd_rn(r, g);
          first = false;
        }
      }
      out[le] = r;
    };
    for (int64_t e = threadIdx.x; e < head; e += blockDim.x) one(e);
    for (int64_t e = body_end + threadIdx.x; e < n; e += blockDim.x) one(e);
  }
  // every owner finished pulling its helpers' staging (and every helper its inputs)
  cross_barrier(s, peer, a.channel, 1, ep);
}

template <int NR, bool BF16, bool MC = false>
__global__ void __launch_bounds__(kThreads) symm_rs_help_kernel(float* __restrict__ out,
                                                                const __grid_constant__ Args a,
                                                                const __grid_constant__ HArgs h,
                                                                const __grid_constant__ Weights wt) {
  set_ctx(blockIdx.x, gridDim.x);
  symm_rs_help_kernel_body<NR, BF16, MC>(out, a, h, wt);
}

// ---------------------------------------------------------------- virtual ranks
//
// All N ranks of one collective as ONE cooperative grid on one GPU (CTA b of
// rank r at blockIdx.x = r * ctas + b, each rank's arguments from device
// memory, the peer table of every rank pointing into one allocation): the
// same kernel bodies and in-kernel barriers as N real launches, with every
// CTA guaranteed co-resident. Test support for the 1-GPU parity runs
// (het_symm_virtual; tests/test_virtual_ranks.py).

struct VRank {
  Args a;
  HArgs h;
  const float* src;
  float* out;
};

enum VKind { kVAg = 0, kVAgHelp = 1, kVRs = 2, kVRs16 = 3, kVRsHelp = 4 };

template <int KIND, int NR, bool BF16>
__global__ void __launch_bounds__(kThreads) symm_virtual_kernel(const VRank* __restrict__ v,
                                                                int ctas,
                                                                const __grid_constant__ Weights wt) {
  const VRank& x = v[blockIdx.x / ctas];
  set_ctx(blockIdx.x % ctas, ctas);
  if constexpr (KIND == kVAg) {
    symm_ag_kernel_body<false, NR>(x.src, x.a);
  } else if constexpr (KIND == kVAgHelp) {
    symm_ag_help_kernel_body<NR>(x.src, x.a, x.h);
  } else if constexpr (KIND == kVRs) {
    symm_rs_kernel_body<false, NR>(x.out, x.a);
  } else if constexpr (KIND == kVRs16) {
    symm_rs_bf16_kernel_body<NR>(x.out, x.a, wt);
  } else {
    symm_rs_help_kernel_body<NR, BF16>(x.out, x.a, x.h, wt);
  }
}

// multicast kernels do not loop over ranks; peer kernels get the rank count
// as a template constant for 2/4/8 ranks so their per-rank loops unroll
#define HET_DISPATCH_NR(mc, n, LAUNCH) \
  do {                                 \
    if (mc) {                          \
      LAUNCH(true, 0);                 \
    } else if ((n) == 2) {             \
      LAUNCH(false, 2);                \
    } else if ((n) == 4) {             \
      LAUNCH(false, 4);                \
    } else if ((n) == 8) {             \
      LAUNCH(false, 8);                \
    } else {                           \
      LAUNCH(false, 0);                \
    }                                  \
  } while (0)

// Per-call route: NVLS multicast costs every GPU S bytes of link traffic
// (the switch loops a GPU's own range back to it), peer push/pull costs
// max((N-1) * max_j s_j, S - min_i s_i). Pick the cheaper one.
bool pick_multicast(const het_symm_t* s, const int64_t* counts, int policy) {
  if (!s->mc_base || policy == HET_SYMM_PEER) return false;
  if (policy == HET_SYMM_MULTICAST) return true;
  int64_t total = 0, mx = 0, mn = INT64_MAX;
  for (int j = 0; j < s->nranks; ++j) {
    total += counts[j];
    mx = counts[j] > mx ? counts[j] : mx;
    mn = counts[j] < mn ? counts[j] : mn;
  }
  const int64_t push = (s->nranks - 1) * mx > total - mn ? (s->nranks - 1) * mx : total - mn;
  return total < push;
}

// Relay pairing for the peer all-gather (HET_SYMM_RELAY). Ranks sorted by
// count, the i-th largest owner A pairs with the i-th smallest B (sB < sA).
// A sends a fraction f of its body to B only and B forwards it to the other
// N-2 ranks. Egress A = sA((N-1) - (N-2) f), egress B = sB(N-1) + (N-2) f sA;
// equal at f = (sA - sB)(N-1) / (2 (N-2) sA). DESIGN.md §5.
void relay_plan(const het_symm_t* s, const int64_t* counts, const int64_t* offsets,
                uint64_t unit_off, Args* a) {
  const int n = s->nranks;
  if (n < 3) return;
  // f is scaled by 1.25 past the egress balance: B's link idles until A's
  // first relay vectors land, so a slightly larger share evens the finish.
  // Sweep 0.5-1.5 at N=4, 1 GB (profiles/r1_final/relay_fscale_n4.jsonl):
  // 2:1 589 -> 616 GB/s, planner 674 -> 686. HET_RELAY_FSCALE overrides.
  static const double fscale = [] {
    const char* e = getenv("HET_RELAY_FSCALE");
    return e ? atof(e) : 1.25;
  }();
  int order[HET_MAX_RANKS];
  for (int j = 0; j < n; ++j) order[j] = j;
  for (int i = 1; i < n; ++i)   // stable insertion sort, count descending
    for (int j = i; j > 0 && counts[order[j]] > counts[order[j - 1]]; --j) {
      const int t = order[j];
      order[j] = order[j - 1];
      order[j - 1] = t;
    }
  for (int i = 0; i < n / 2; ++i) {
    const int A = order[i], B = order[n - 1 - i];
    const int64_t sa = counts[A], sb = counts[B];
    if (sa <= sb) break;
    double f = fscale * static_cast<double>(sa - sb) * (n - 1) / (2.0 * (n - 2) * sa);
    if (f > 1.0) f = 1.0;
    int64_t h1, h2, nvec;
    ag_geometry(unit_off + static_cast<uint64_t>(offsets[A]) * 2, sa, &h1, &h2, &nvec);
    const int64_t rv = static_cast<int64_t>(f * static_cast<double>(nvec));
    if (rv <= 0) continue;
    if (s->rank == A) {
      a->relay_to = B;
      a->relay_vecs = rv;
    }
    if (s->rank == B) {
      a->relay_from = A;
      a->from_count = sa;
      a->from_offset = offsets[A];
      a->from_vecs = rv;
    }
  }
}


// Helper plan (HET_SYMM_HELPERS), computed identically on every rank from the
// shard table. Link cost per element (bytes), for a rank's own range split
// into a direct part d and helper pieces r = s - d:
//   owner:  alpha * d + beta * r      (AG: (N-1) d + r egress;  RS fp32:
//                                      (N-1) d + r ingress; RS bf16 wire:
//                                      2(N-1) d + 4 r ingress)
//   helper: alpha * s_h + gamma * a   (a = elements it relays; AG gamma = N-2
//                                      forwards, RS gamma = (N-1) pulls x ES)
// Binary search for the smallest per-link load T such that the heavy ranks'
// excess fits into the light ranks' spare capacity, then fill: heavy owners in
// count order (largest first), helpers lightest first. Pieces are in units of
// the owner's body vectors (vnec[i] of them); the direct part takes the head.
struct HelperPlan {
  int npieces = 0;
  int owner[2 * HET_MAX_RANKS], helper[2 * HET_MAX_RANKS];
  int64_t lo[2 * HET_MAX_RANKS], hi[2 * HET_MAX_RANKS];
  int64_t direct[HET_MAX_RANKS];
};

HelperPlan helper_plan(int n, const int64_t* counts, const int64_t* nvecs, double alpha,
                       double beta, double gamma) {
  HelperPlan hp;
  for (int i = 0; i < n; ++i) hp.direct[i] = nvecs[i];
  if (n < 3 || alpha <= beta) return hp;
  double mx = 0;
  for (int i = 0; i < n; ++i) mx = counts[i] > mx ? static_cast<double>(counts[i]) : mx;
  auto excess = [&](double T, int i) {       // elements owner i must relay at load T
    const double c = static_cast<double>(counts[i]);
    if (alpha * c <= T) return 0.0;
    double d = (T - beta * c) / (alpha - beta);
    if (d < 0) d = 0;
    return c - d;
  };
  auto spare = [&](double T, int j) {
    const double c = static_cast<double>(counts[j]);
    return alpha * c < T ? (T - alpha * c) / gamma : 0.0;
  };
  auto feasible = [&](double T) {
    double need = 0, have = 0;
    for (int i = 0; i < n; ++i) {
      if (beta * counts[i] > T) return false;
      need += excess(T, i);
      have += spare(T, i);
    }
    return need <= have;
  };
  double lo = 0, hi = alpha * mx;
  if (hi <= 0) return hp;
  for (int it = 0; it < 60; ++it) {
    const double mid = 0.5 * (lo + hi);
    (feasible(mid) ? hi : lo) = mid;
  }
  const double T = hi;
  int order[HET_MAX_RANKS];
  for (int j = 0; j < n; ++j) order[j] = j;
  for (int i = 1; i < n; ++i)      // stable insertion sort, count descending
    for (int j = i; j > 0 && counts[order[j]] > counts[order[j - 1]]; --j) {
      const int t = order[j];
      order[j] = order[j - 1];
      order[j - 1] = t;
    }
  // helpers: ranks with spare capacity at T and nothing to relay, lightest first
  int helpers[HET_MAX_RANKS], nh = 0;
  double cap[HET_MAX_RANKS];
  for (int oi = n - 1; oi >= 0; --oi) {
    const int j = order[oi];
    cap[j] = spare(T, j);
    if (cap[j] > 0 && excess(T, j) <= 0) helpers[nh++] = j;
  }
  int hk = 0;
  for (int oi = 0; oi < n; ++oi) {
    const int i = order[oi];
    const double ex = excess(T, i);
    if (ex <= 0 || nvecs[i] <= 0 || hk >= nh) continue;
    const double per_vec = static_cast<double>(counts[i]) / static_cast<double>(nvecs[i]);
    int64_t rv = static_cast<int64_t>(ex / per_vec + 0.5);
    if (rv > nvecs[i]) rv = nvecs[i];
    if (rv <= 0) continue;
    hp.direct[i] = nvecs[i] - rv;
    int64_t pos = hp.direct[i];
    int last = -1;
    while (pos < nvecs[i] && hk < nh && hp.npieces < 2 * HET_MAX_RANKS) {
      const int h = helpers[hk];
      int64_t take = static_cast<int64_t>(cap[h] / per_vec + 0.5);
      if (take < 1) take = 1;
      if (take > nvecs[i] - pos || hk == nh - 1) take = nvecs[i] - pos;
      last = hp.npieces++;
      hp.owner[last] = i;
      hp.helper[last] = h;
      hp.lo[last] = pos;
      hp.hi[last] = pos + take;
      pos += take;
      cap[h] -= static_cast<double>(take) * per_vec;
      if (cap[h] <= 0.5 * per_vec) ++hk;
    }
    if (pos < nvecs[i]) {     // out of piece slots: the rest rides on the last piece
      if (last >= 0) hp.hi[last] = nvecs[i];
      else hp.direct[i] = nvecs[i];
    }
  }
  return hp;
}

// Fill this rank's role tables from the plan.
void fill_hargs(const HelperPlan& hp, int rank, const int64_t* counts, const int64_t* offsets,
                int ctas, HArgs* h) {
  std::memset(h, 0, sizeof(*h));
  h->direct = hp.direct[rank];
  int64_t kmax = 1;
  const int64_t per_iter = static_cast<int64_t>(ctas) * kThreads * kUnroll;
  for (int k = 0; k < hp.npieces; ++k) {
    const int64_t it = (hp.hi[k] - hp.lo[k] + per_iter - 1) / per_iter;
    kmax = it > kmax ? it : kmax;
    if (hp.owner[k] == rank && h->n_own < HET_MAX_RANKS) {
      const int j = h->n_own++;
      h->own_peer[j] = hp.helper[k];
      h->own_lo[j] = hp.lo[k];
      h->own_hi[j] = hp.hi[k];
    }
    if (hp.helper[k] == rank && h->n_help < HET_MAX_RANKS) {
      const int j = h->n_help++;
      h->help_peer[j] = hp.owner[k];
      h->help_lo[j] = hp.lo[k];
      h->help_hi[j] = hp.hi[k];
      h->help_count[j] = counts[hp.owner[k]];
      h->help_offset[j] = offsets[hp.owner[k]];
    }
  }
  // iterations per progress signal: at most 4000 signals (the epoch * 4096 + k
  // encoding); HET_HELPER_GRAN forces a coarser hand-off for measurement sweeps
  static const int forced = [] {
    const char* e = getenv("HET_HELPER_GRAN");
    return e ? atoi(e) : 0;
  }();
  // Default 4 iterations per hand-off: every signal drains the CTA's remote
  // stores (release fence), and per-iteration signals held the single-owner AG
  // at N=4 to 421 GB/s against 627 with 4 (profiles/r2/helpers_c128_g*.jsonl).
  const int64_t fine = (kmax + 3999) / 4000;
  const int64_t want = forced > 0 ? forced : 4;
  h->gran = static_cast<int>(want > fine ? want : fine);
}

// Body-vector counts of every rank's range (AG: bf16 at unit_off; RS: fp32 or
// bf16 at data_off), the geometry the kernels derive on the device.
void body_vectors(int op, int n, const int64_t* counts, const int64_t* offsets, uint64_t off,
                  int64_t* nvecs) {
  for (int j = 0; j < n; ++j) {
    if (op == HET_OP_AG) {
      int64_t h1, h2, nv;
      ag_geometry(off + static_cast<uint64_t>(offsets[j]) * 2, counts[j], &h1, &h2, &nv);
      nvecs[j] = nv;
    } else {             // RS, RS_MC: fp32; RS_BF16: bf16
      const int es = op == HET_OP_RS_BF16 ? 2 : 4;
      const uint64_t src0 = off + static_cast<uint64_t>(offsets[j]) * es;
      int64_t hd = static_cast<int64_t>(((16 - (src0 & 15)) & 15) / es);
      if (hd > counts[j]) hd = counts[j];
      nvecs[j] = (counts[j] - hd) / (16 / es);
    }
  }
}

// Per-element link costs in bytes (alpha, beta, gamma) of helper_plan for an op at n ranks.
void helper_costs(int op, int n, double* alpha, double* beta, double* gamma) {
  if (op == HET_OP_AG) {
    *alpha = 2.0 * (n - 1); *beta = 2; *gamma = 2.0 * (n - 2);
  } else if (op == HET_OP_RS) {
    *alpha = 4.0 * (n - 1); *beta = 4; *gamma = 4.0 * (n - 1);
  } else if (op == HET_OP_RS_MC) {
    // the owner's direct part and the helpers' pieces arrive as one stream of
    // switch-reduced sums (4 B per element) at MC_EFF = 0.83 of a peer stream's
    // rate (hetstep.py), the staged sums as a plain pull: peer-equivalent bytes
    *alpha = 4.0 / 0.83; *beta = 4; *gamma = 4.0 / 0.83;
  } else {
    *alpha = 2.0 * (n - 1); *beta = 4; *gamma = 2.0 * (n - 1);
  }
}

HelperPlan plan_for(int op, int n, const int64_t* counts, const int64_t* offsets, uint64_t off) {
  int64_t nv[HET_MAX_RANKS];
  body_vectors(op, n, counts, offsets, off, nv);
  double a, b, g;
  helper_costs(op, n, &a, &b, &g);
  return helper_plan(n, counts, nv, a, b, g);
}

int check_symm(const het_symm_t* s, const int64_t* counts, const int64_t* offsets, int ctas) {
  if (!s || s->nranks < 1 || s->nranks > HET_MAX_RANKS || s->rank < 0 || s->rank >= s->nranks)
    return fail(HET_EARG, "het_symm: bad rank table");
  if (!counts || !offsets) return fail(HET_EARG, "het_symm: null shard table");
  if (ctas < 1 || ctas > kMaxCtas) return fail(HET_EARG, "het_symm: ctas must be 1..%d", kMaxCtas);
  int64_t pos = 0;
  for (int j = 0; j < s->nranks; ++j) {
    if (counts[j] < 0 || offsets[j] != pos)
      return fail(HET_EARG, "het_symm: shard table not contiguous at rank %d", j);
    pos += counts[j];
  }
  for (int j = 0; j < s->nranks; ++j)
    if (!s->peer_base[j]) return fail(HET_EARG, "het_symm: missing peer base %d", j);
  return HET_OK;
}

}  // namespace

namespace het {
int set_symm_timeout_ms(int ms) {
  if (ms < 1) return fail(HET_EARG, "het_tune: symmetric barrier timeout must be >= 1 ms");
  g_spin_timeout_ns = static_cast<uint64_t>(ms) * 1000ull * 1000ull;
  return HET_OK;
}
}  // namespace het

extern "C" {

int64_t het_symm_signal_bytes(void) {
  return static_cast<int64_t>(slot_bytes()) + 256;   // + the device epoch bases
}

static int epoch_update(const het_symm_t* s, int channel, uint32_t v, int add, void* stream,
                        const char* who) {
  if (!s || s->rank < 0 || s->rank >= s->nranks || s->nranks > HET_MAX_RANKS)
    return fail(HET_EARG, "%s: bad descriptor", who);
  if (channel < 0 || channel >= HET_SYMM_CHANNELS) return fail(HET_EARG, "%s: bad channel", who);
  uint32_t* b = reinterpret_cast<uint32_t*>(s->peer_base[s->rank] + s->signal_off +
                                            slot_bytes()) + channel;
  epoch_update_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(b, v, add);
  return het::check_launch(who);
}

int het_symm_epoch_set(const het_symm_t* s, int channel, uint32_t value, void* stream) {
  return epoch_update(s, channel, value, 0, stream, "het_symm_epoch_set");
}

int het_symm_epoch_add(const het_symm_t* s, int channel, uint32_t delta, void* stream) {
  return epoch_update(s, channel, delta, 1, stream, "het_symm_epoch_add");
}

int het_symm_status(int reset) {
  int v = 0;
  if (cudaMemcpyFromSymbol(&v, g_symm_status, sizeof(int)) != cudaSuccess)
    return fail(HET_ECUDA, "het_symm_status: %s", cudaGetErrorString(cudaGetLastError()));
  if (reset) {
    const int z = 0;
    cudaMemcpyToSymbol(g_symm_status, &z, sizeof(int));
  }
  return v;
}

int het_symm_helper_plan(int op, int nranks, const int64_t* counts, const int64_t* offsets,
                         uint64_t off, int64_t* out_direct, int32_t* out_pieces, int max_pieces,
                         double* link_load) {
  if (nranks < 1 || nranks > HET_MAX_RANKS || !counts || !offsets ||
      (op != HET_OP_AG && op != HET_OP_RS && op != HET_OP_RS_BF16 && op != HET_OP_RS_MC))
    return -fail(HET_EARG, "het_symm_helper_plan: bad args");
  const HelperPlan hp = plan_for(op, nranks, counts, offsets, off);
  if (out_direct)
    for (int j = 0; j < nranks; ++j) out_direct[j] = hp.direct[j];
  if (out_pieces)
    for (int k = 0; k < hp.npieces && k < max_pieces; ++k) {
      out_pieces[2 * k] = hp.owner[k];
      out_pieces[2 * k + 1] = hp.helper[k];
    }
  if (link_load) {       // per-rank link bytes of this plan (AG egress / RS ingress)
    int64_t nv[HET_MAX_RANKS];
    body_vectors(op, nranks, counts, offsets, off, nv);
    double a, b, g;
    helper_costs(op, nranks, &a, &b, &g);
    for (int j = 0; j < nranks; ++j) {
      const double per = nv[j] > 0 ? static_cast<double>(counts[j]) / nv[j] : 0.0;
      link_load[j] = a * (counts[j] - (nv[j] - hp.direct[j]) * per);
    }
    for (int k = 0; k < hp.npieces; ++k) {
      const int i = hp.owner[k], h = hp.helper[k];
      const double el = static_cast<double>(hp.hi[k] - hp.lo[k]) * counts[i] / nv[i];
      link_load[i] += b * el;
      link_load[h] += g * el;
    }
  }
  return hp.npieces;
}

int het_symm_virtual(int op, int nranks, const het_symm_t* descs, const float* const* srcs,
                     float* const* outs, const int64_t* counts, const int64_t* offsets,
                     uint64_t off, const float* weights, uint32_t epoch, int channel,
                     int end_barrier, int policy, uint64_t stage_off, int ctas, void* stream) {
  if (!descs || nranks < 1 || nranks > HET_MAX_RANKS || !srcs || !outs ||
      (op != HET_OP_AG && op != HET_OP_RS && op != HET_OP_RS_BF16))
    return fail(HET_EARG, "het_symm_virtual: bad args");
  if (channel < 0 || channel >= HET_SYMM_CHANNELS) return fail(HET_EARG, "bad channel");
  if (off & 15) return fail(HET_EARG, "het_symm_virtual: offset not 16B aligned");
  if (op != HET_OP_AG && policy == HET_SYMM_RELAY) policy = HET_SYMM_AUTO;
  if (policy == HET_SYMM_HELPERS_MC) policy = HET_SYMM_HELPERS;   // one GPU: no multicast
  const bool helpers = policy == HET_SYMM_HELPERS;
  if (op == HET_OP_RS_BF16 && (!weights || (helpers && (stage_off & 15))))
    return fail(HET_EARG, "het_symm_virtual: bf16 wire needs weights (and a 16B stage)");
  VRank host[HET_MAX_RANKS];
  HelperPlan hp;
  if (helpers) hp = plan_for(op, nranks, counts, offsets, off);
  for (int r = 0; r < nranks; ++r) {
    const het_symm_t* d = &descs[r];
    int rc = check_symm(d, counts, offsets, ctas);
    if (rc != HET_OK) return rc;
    if (d->nranks != nranks || d->rank != r || d->mc_base)
      return fail(HET_EARG, "het_symm_virtual: descriptor %d is not rank %d of %d (no multicast)",
                  r, r, nranks);
    std::memset(&host[r], 0, sizeof(VRank));
    Args a{*d, off, counts[r], offsets[r], epoch, channel, op == HET_OP_AG ? 1 : end_barrier,
           -1, -1, 0, 0, 0, 0, g_spin_timeout_ns};
    if (op == HET_OP_AG && policy == HET_SYMM_RELAY) relay_plan(d, counts, offsets, off, &a);
    host[r].a = a;
    if (helpers) {
      fill_hargs(hp, r, counts, offsets, ctas, &host[r].h);
      host[r].h.stage_off = op == HET_OP_RS_BF16 ? stage_off : off;
    }
    host[r].src = srcs[r];
    host[r].out = outs[r];
  }
  Weights wt{};
  if (weights)
    for (int j = 0; j < nranks; ++j) wt.w[j] = weights[j];
  const int kind = op == HET_OP_AG ? (helpers ? kVAgHelp : kVAg)
                                   : (helpers ? kVRsHelp : (op == HET_OP_RS ? kVRs : kVRs16));
  const bool bf16 = op == HET_OP_RS_BF16;
  void* kern = nullptr;
#define HET_VK(K, NRV, B) reinterpret_cast<void*>(symm_virtual_kernel<K, NRV, B>)
#define HET_VK_NR(K, B)                                                              \
  (nranks == 2 ? HET_VK(K, 2, B) : nranks == 4 ? HET_VK(K, 4, B)                     \
   : nranks == 8 ? HET_VK(K, 8, B) : HET_VK(K, 0, B))
  switch (kind) {
    case kVAg: kern = HET_VK_NR(kVAg, false); break;
    case kVAgHelp: kern = HET_VK_NR(kVAgHelp, false); break;
    case kVRs: kern = HET_VK_NR(kVRs, false); break;
    case kVRs16: kern = HET_VK_NR(kVRs16, false); break;
    default: kern = bf16 ? HET_VK_NR(kVRsHelp, true) : HET_VK_NR(kVRsHelp, false);
  }
#undef HET_VK_NR
#undef HET_VK
  // every CTA of the grid must be co-resident: refuse instead of risking a wait
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, 0);
  const int grid = nranks * ctas;
  if (grid > per_sm * sms)
    return fail(HET_EARG, "het_symm_virtual: %d CTAs exceed the %d co-resident (%d per SM)",
                grid, per_sm * sms, per_sm);
  VRank* dv = nullptr;
  if (cudaMalloc(&dv, sizeof(VRank) * nranks) != cudaSuccess)
    return fail(HET_ECUDA, "het_symm_virtual: %s", cudaGetErrorString(cudaGetLastError()));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(dv, host, sizeof(VRank) * nranks, cudaMemcpyHostToDevice, st);
  int c = ctas;
  void* args[] = {&dv, &c, &wt};
  if (e == cudaSuccess)
    e = cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kThreads), args, 0, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);   // test support: synchronous
  cudaFree(dv);
  if (e != cudaSuccess) return fail(HET_ECUDA, "het_symm_virtual: %s", cudaGetErrorString(e));
  return HET_OK;
}

int het_symm_status_async(int32_t* dst, void* stream) {
  if (!dst) return fail(HET_EARG, "het_symm_status_async: null dst");
  status_copy_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(dst);
  return het::check_launch("het_symm_status_async");
}

int het_symm_allgather_pack(const het_symm_t* s, const float* src, uint64_t unit_off,
                            const int64_t* counts, const int64_t* offsets, uint32_t epoch,
                            int channel, int policy, int ctas, void* stream) {
  int rc = check_symm(s, counts, offsets, ctas);
  if (rc != HET_OK) return rc;
  if (channel < 0 || channel >= HET_SYMM_CHANNELS) return fail(HET_EARG, "bad channel");
  if (counts[s->rank] > 0 && !src) return fail(HET_EARG, "het_symm_allgather_pack: null src");
  if (unit_off & 15) return fail(HET_EARG, "het_symm_allgather_pack: unit offset not 16B aligned");
  if (policy == HET_SYMM_HELPERS_MC) policy = HET_SYMM_HELPERS;
  Args a{*s, unit_off, counts[s->rank], offsets[s->rank], epoch, channel, 1, -1, -1, 0, 0, 0, 0,
         g_spin_timeout_ns};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (policy == HET_SYMM_HELPERS) {
    HArgs h;
    fill_hargs(plan_for(HET_OP_AG, s->nranks, counts, offsets, unit_off), s->rank, counts,
               offsets, ctas, &h);
    switch (s->nranks) {
      case 2: symm_ag_help_kernel<2><<<ctas, kThreads, 0, st>>>(src, a, h); break;
      case 4: symm_ag_help_kernel<4><<<ctas, kThreads, 0, st>>>(src, a, h); break;
      case 8: symm_ag_help_kernel<8><<<ctas, kThreads, 0, st>>>(src, a, h); break;
      default: symm_ag_help_kernel<0><<<ctas, kThreads, 0, st>>>(src, a, h);
    }
    return het::check_launch("het_symm_allgather_pack");
  }
  const bool mc = policy == HET_SYMM_RELAY ? false : pick_multicast(s, counts, policy);
  if (policy == HET_SYMM_RELAY) relay_plan(s, counts, offsets, unit_off, &a);
#define HET_AG(MCV, NRV) symm_ag_kernel<MCV, NRV><<<ctas, kThreads, 0, st>>>(src, a)
  HET_DISPATCH_NR(mc, s->nranks, HET_AG);
#undef HET_AG
  return het::check_launch("het_symm_allgather_pack");
}

int het_symm_reduce_scatter(const het_symm_t* s, uint64_t acc_off, float* out,
                            const int64_t* counts, const int64_t* offsets, uint32_t epoch,
                            int channel, int end_barrier, int policy, int ctas, void* stream) {
  int rc = check_symm(s, counts, offsets, ctas);
  if (rc != HET_OK) return rc;
  if (channel < 0 || channel >= HET_SYMM_CHANNELS) return fail(HET_EARG, "bad channel");
  if (counts[s->rank] > 0 && !out) return fail(HET_EARG, "het_symm_reduce_scatter: null out");
  if (acc_off & 15) return fail(HET_EARG, "het_symm_reduce_scatter: acc offset not 16B aligned");
  Args a{*s, acc_off, counts[s->rank], offsets[s->rank], epoch, channel, end_barrier};
  a.timeout_ns = g_spin_timeout_ns;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (policy == HET_SYMM_HELPERS_MC && !s->mc_base) policy = HET_SYMM_HELPERS;
  if (policy == HET_SYMM_HELPERS_MC) {    // helpers reduce their pieces in the switch
    HArgs h;
    fill_hargs(plan_for(HET_OP_RS_MC, s->nranks, counts, offsets, acc_off), s->rank, counts,
               offsets, ctas, &h);
    h.stage_off = acc_off;
    Weights wt{};
    switch (s->nranks) {
      case 2: symm_rs_help_kernel<2, false, true><<<ctas, kThreads, 0, st>>>(out, a, h, wt); break;
      case 4: symm_rs_help_kernel<4, false, true><<<ctas, kThreads, 0, st>>>(out, a, h, wt); break;
      case 8: symm_rs_help_kernel<8, false, true><<<ctas, kThreads, 0, st>>>(out, a, h, wt); break;
      default: symm_rs_help_kernel<0, false, true><<<ctas, kThreads, 0, st>>>(out, a, h, wt);
    }
    return het::check_launch("het_symm_reduce_scatter");
  }
  if (policy == HET_SYMM_HELPERS) {       // helpers reduce in place in their own acc
    HArgs h;
    fill_hargs(plan_for(HET_OP_RS, s->nranks, counts, offsets, acc_off), s->rank, counts,
               offsets, ctas, &h);
    h.stage_off = acc_off;
    Weights wt{};
    switch (s->nranks) {
      case 2: symm_rs_help_kernel<2, false><<<ctas, kThreads, 0, st>>>(out, a, h, wt); break;
      case 4: symm_rs_help_kernel<4, false><<<ctas, kThreads, 0, st>>>(out, a, h, wt); break;
      case 8: symm_rs_help_kernel<8, false><<<ctas, kThreads, 0, st>>>(out, a, h, wt); break;
      default: symm_rs_help_kernel<0, false><<<ctas, kThreads, 0, st>>>(out, a, h, wt);
    }
    return het::check_launch("het_symm_reduce_scatter");
  }
  const bool mc = pick_multicast(s, counts, policy);
#define HET_RS(MCV, NRV) symm_rs_kernel<MCV, NRV><<<ctas, kThreads, 0, st>>>(out, a)
  HET_DISPATCH_NR(mc, s->nranks, HET_RS);
#undef HET_RS
  return het::check_launch("het_symm_reduce_scatter");
}

int het_symm_reduce_scatter_bf16(const het_symm_t* s, uint64_t grad_off, float* out,
                                 const int64_t* counts, const int64_t* offsets,
                                 const float* weights, uint32_t epoch, int channel,
                                 int end_barrier, int policy, uint64_t stage_off, int ctas,
                                 void* stream) {
  int rc = check_symm(s, counts, offsets, ctas);
  if (rc != HET_OK) return rc;
  if (channel < 0 || channel >= HET_SYMM_CHANNELS) return fail(HET_EARG, "bad channel");
  if (!weights) return fail(HET_EARG, "het_symm_reduce_scatter_bf16: null weights");
  if (counts[s->rank] > 0 && !out) return fail(HET_EARG, "het_symm_reduce_scatter_bf16: null out");
  if (grad_off & 15) return fail(HET_EARG, "het_symm_reduce_scatter_bf16: grad offset not 16B aligned");
  if (policy == HET_SYMM_HELPERS_MC) policy = HET_SYMM_HELPERS;   // weights: no switch sum
  Args a{*s, grad_off, counts[s->rank], offsets[s->rank], epoch, channel, end_barrier};
  a.timeout_ns = g_spin_timeout_ns;
  Weights wt{};
  for (int j = 0; j < s->nranks; ++j) wt.w[j] = weights[j];
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (policy == HET_SYMM_HELPERS) {       // helpers stage fp32 sums at stage_off
    if (stage_off & 15)
      return fail(HET_EARG, "het_symm_reduce_scatter_bf16: stage offset not 16B aligned");
    HArgs h;
    fill_hargs(plan_for(HET_OP_RS_BF16, s->nranks, counts, offsets, grad_off), s->rank, counts,
               offsets, ctas, &h);
    h.stage_off = stage_off;
    switch (s->nranks) {
      case 2: symm_rs_help_kernel<2, true><<<ctas, kThreads, 0, st>>>(out, a, h, wt); break;
      case 4: symm_rs_help_kernel<4, true><<<ctas, kThreads, 0, st>>>(out, a, h, wt); break;
      case 8: symm_rs_help_kernel<8, true><<<ctas, kThreads, 0, st>>>(out, a, h, wt); break;
      default: symm_rs_help_kernel<0, true><<<ctas, kThreads, 0, st>>>(out, a, h, wt);
    }
    return het::check_launch("het_symm_reduce_scatter_bf16");
  }
  switch (s->nranks) {
    case 2: symm_rs_bf16_kernel<2><<<ctas, kThreads, 0, st>>>(out, a, wt); break;
    case 4: symm_rs_bf16_kernel<4><<<ctas, kThreads, 0, st>>>(out, a, wt); break;
    case 8: symm_rs_bf16_kernel<8><<<ctas, kThreads, 0, st>>>(out, a, wt); break;
    default: symm_rs_bf16_kernel<0><<<ctas, kThreads, 0, st>>>(out, a, wt);
  }
  return het::check_launch("het_symm_reduce_scatter_bf16");
}

}  // extern "C"

// sm_100a streaming kernels of the uneven-FSDP train step.
//
// All four are HBM-bound elementwise passes (no data reuse, no tensor-core
// work — see DESIGN.md "Kernels"): the design levers are 16-byte vector
// accesses, several independent 16-byte requests in flight per thread
// (loads issued before use), and a grid sized in multiples of the 148 SMs
// with a grid-stride loop. Inputs touched once are loaded with the
// streaming/evict-first hint so they do not displace the next unit's
// gathered parameters in the 126 MB L2.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "hetstep.h"
#include "hetstep_internal.cuh"

namespace het {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HET_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return HET_OK;
}

int g_sm_budget = 0;   // het_tune(HET_TUNE_SM_BUDGET); 0 = the whole device
int g_acc_grid = 0;    // het_tune(HET_TUNE_ACC_GRID): 0 persistent, 1 one CTA per chunk

int sm_count() {
  static int dev_sms = 0;
  if (dev_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, dev);
    if (dev_sms <= 0) dev_sms = 148;
  }
  return g_sm_budget > 0 && g_sm_budget < dev_sms ? g_sm_budget : dev_sms;
}

int grid_for(int64_t work_items, int threads) {
  const int sms = sm_count();
  int64_t need = (work_items + threads - 1) / threads;
  int64_t cap = static_cast<int64_t>(sms) * 8;  // 8 x 256-thread CTAs resident per SM
  if (need < 1) need = 1;
  return static_cast<int>(need < cap ? need : cap);
}

}  // namespace het

using het::fail;

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ float bf16_bits_to_f32(uint32_t bits16) {
  return __uint_as_float(bits16 << 16);
}

__device__ __forceinline__ void unpack8(const uint4& raw, float (&f)[8]) {
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = bf16_bits_to_f32(w[i] & 0xffffu);
    f[2 * i + 1] = bf16_bits_to_f32(w[i] >> 16);
  }
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// 256-bit global accesses (sm_100: LDG/STG.E.ENL2.256): one instruction per
// 8 fp32, half the memory instructions of float4 at the same bytes in flight.
struct F8 {
  float x[8];
};

__device__ __forceinline__ F8 ld8(const float* a) {
  F8 r;
  asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]),
                 "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7])
               : "l"(a));
  return r;
}

__device__ __forceinline__ F8 ld8_stream(const float* a) {   // touch-once input
  F8 r;
  asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]),
                 "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7])
               : "l"(a));
  return r;
}

__device__ __forceinline__ void st8(float* a, const F8& r) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(a), "f"(r.x[0]),
               "f"(r.x[1]), "f"(r.x[2]), "f"(r.x[3]), "f"(r.x[4]), "f"(r.x[5]), "f"(r.x[6]),
               "f"(r.x[7])
               : "memory");
}

__host__ __device__ __forceinline__ bool aligned32(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 31) == 0;
}

// ---------------------------------------------------------------- pack

__global__ void __launch_bounds__(kThreads) pack_vec_kernel(const float4* __restrict__ src,
                                                            uint2* __restrict__ dst,
                                                            int64_t n4) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += 2 * stride) {
    const bool two = i + stride < n4;
    float4 a = __ldcs(src + i);
    float4 b = two ? __ldcs(src + i + stride) : make_float4(0.f, 0.f, 0.f, 0.f);
    dst[i] = make_uint2(pack2(a.x, a.y), pack2(a.z, a.w));
    if (two) dst[i + stride] = make_uint2(pack2(b.x, b.y), pack2(b.z, b.w));
  }
}

__global__ void pack_scalar_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                   int64_t n) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    dst[i] = __float2bfloat16_rn(src[i]);
}

// ---------------------------------------------------------------- accumulate

struct SegTable {
  het_seg_t seg[HET_MAX_SEGS];
  int64_t first_block[HET_MAX_SEGS + 1];  // prefix sum of blocks per segment
  int nseg;
};

constexpr int kAccVec = 8;                 // bf16 elements per 16-byte load
// (THREADS, ITERS) variants: ITERS 16-byte gradient loads in flight per thread;
// a CTA covers THREADS * 8 * ITERS elements of one segment.
struct AccShape {
  int threads, iters;
};
constexpr AccShape kAccShapes[] = {{256, 4}, {256, 2}, {256, 1}, {512, 2}, {512, 1}, {128, 4}};
int g_acc_variant = 4;   // het_tune(HET_TUNE_ACC_VARIANT, i); 4 = (512 threads, 1 load) measured best

template <int MODE>
__device__ __forceinline__ float acc_op(float a, float g, float w) {
  return MODE == HET_ACC_FIRST ? w * g : fmaf(w, g, a);
}

// One chunk (THREADS * 8 * ITERS elements) of one segment.
template <int MODE, int THREADS, int ITERS>
__device__ __forceinline__ void acc_chunk(float* __restrict__ acc, const het_seg_t& sg,
                                          int64_t base, float w) {
  constexpr int64_t kAccChunk = static_cast<int64_t>(THREADS) * kAccVec * ITERS;
  const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(sg.src);
  float* dst = acc + sg.dst_off;
  const bool vec_ok = ((reinterpret_cast<uintptr_t>(src) & 15) == 0) &&
                      ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
  if (vec_ok && base + kAccChunk <= sg.n) {
    uint4 raw[ITERS];
    F8 a[ITERS];
    const bool wide = aligned32(dst);     // 256-bit accumulator accesses
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t e = base + (static_cast<int64_t>(it) * THREADS + threadIdx.x) * kAccVec;
      raw[it] = __ldcs(reinterpret_cast<const uint4*>(src + e));
      if (MODE == HET_ACC_FIRST) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[it].x[k] = 0.f;
      } else if (wide) {
        a[it] = ld8(dst + e);
      } else {
        const float4 lo = *reinterpret_cast<const float4*>(dst + e);
        const float4 hi = *reinterpret_cast<const float4*>(dst + e + 4);
        a[it] = F8{{lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w}};
      }
    }
#pragma unroll
    for (int it = 0; it < ITERS; ++it) {
      const int64_t e = base + (static_cast<int64_t>(it) * THREADS + threadIdx.x) * kAccVec;
      float g[8];
      unpack8(raw[it], g);
      F8 o;
#pragma unroll
      for (int k = 0; k < 8; ++k) o.x[k] = acc_op<MODE>(a[it].x[k], g[k], w);
      if (wide) {
        st8(dst + e, o);
      } else {
        *reinterpret_cast<float4*>(dst + e) = make_float4(o.x[0], o.x[1], o.x[2], o.x[3]);
        *reinterpret_cast<float4*>(dst + e + 4) = make_float4(o.x[4], o.x[5], o.x[6], o.x[7]);
      }
    }
    return;
  }
  // ragged tail of a segment (or unaligned segment): scalar, coalesced
  const int64_t end = base + kAccChunk < sg.n ? base + kAccChunk : sg.n;
  for (int64_t e = base + threadIdx.x; e < end; e += THREADS) {
    const float g = __bfloat162float(src[e]);
    const float a = (MODE & HET_ACC_FIRST) ? 0.f : dst[e];
    dst[e] = acc_op<MODE>(a, g, w);
  }
}

// Persistent grid over the launch's chunks (prefix sums in the parameter
// table): a CTA binary-searches its first chunk's segment once, then walks
// forward with the grid stride, so the table lookup is amortised over the
// CTA's chunks instead of paid per chunk.
template <int MODE, int THREADS, int ITERS>
__global__ void __launch_bounds__(THREADS) accumulate_kernel(float* __restrict__ acc,
                                                             const __grid_constant__ SegTable t,
                                                             float w) {
  constexpr int64_t kAccChunk = static_cast<int64_t>(THREADS) * kAccVec * ITERS;
  const int64_t total = t.first_block[t.nseg];
  int64_t b = blockIdx.x;
  if (b >= total) return;
  int lo = 0, hi = t.nseg - 1;            // invariant: first_block[lo] <= b
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (t.first_block[mid] <= b) lo = mid; else hi = mid - 1;
  }
  int s = lo;
  for (; b < total; b += gridDim.x) {
    while (s + 1 < t.nseg && t.first_block[s + 1] <= b) ++s;
    acc_chunk<MODE, THREADS, ITERS>(acc, t.seg[s], (b - t.first_block[s]) * kAccChunk, w);
  }
}

// Several microbatches' gradients of the same segments in one pass (layered
// GA with l_i > 1): source 0 comes from the SegTable, sources 1..NSRC-1 from
// `more`. All NSRC gradient loads (and the acc load) are issued before the
// arithmetic, which runs in microbatch order in registers, so the result is
// bit-identical to NSRC sequential accumulate_kernel passes.
struct MoreSrc {
  const void* src[HET_MAX_ACC_SRC - 1][HET_MAX_SEGS];
};

template <int MODE, int NSRC>
__global__ void __launch_bounds__(512) accumulate_multi_kernel(float* __restrict__ acc,
                                                               const __grid_constant__ SegTable t,
                                                               const __grid_constant__ MoreSrc ms,
                                                               float w) {
  constexpr int64_t kChunk = 512 * kAccVec;
  const int64_t total = t.first_block[t.nseg];
  int64_t b = blockIdx.x;
  if (b >= total) return;
  int lo = 0, hi = t.nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (t.first_block[mid] <= b) lo = mid; else hi = mid - 1;
  }
  int s = lo;
  for (; b < total; b += gridDim.x) {
    while (s + 1 < t.nseg && t.first_block[s + 1] <= b) ++s;
    const het_seg_t& sg = t.seg[s];
    const int64_t base = (b - t.first_block[s]) * kChunk;
    const __nv_bfloat16* src[NSRC];
    src[0] = static_cast<const __nv_bfloat16*>(sg.src);
    uintptr_t bits = reinterpret_cast<uintptr_t>(src[0]);
#pragma unroll
    for (int j = 1; j < NSRC; ++j) {
      src[j] = static_cast<const __nv_bfloat16*>(ms.src[j - 1][s]);
      bits |= reinterpret_cast<uintptr_t>(src[j]);
    }
    float* dst = acc + sg.dst_off;
    if (((bits | reinterpret_cast<uintptr_t>(dst)) & 15) == 0 && base + kChunk <= sg.n) {
      const int64_t e = base + threadIdx.x * kAccVec;
      uint4 raw[NSRC];
#pragma unroll
      for (int j = 0; j < NSRC; ++j) raw[j] = __ldcs(reinterpret_cast<const uint4*>(src[j] + e));
      const bool wide = aligned32(dst);
      F8 a;
      if (MODE == HET_ACC_FIRST) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a.x[k] = 0.f;
      } else if (wide) {
        a = ld8(dst + e);
      } else {
        const float4 lo4 = *reinterpret_cast<const float4*>(dst + e);
        const float4 hi4 = *reinterpret_cast<const float4*>(dst + e + 4);
        a = F8{{lo4.x, lo4.y, lo4.z, lo4.w, hi4.x, hi4.y, hi4.z, hi4.w}};
      }
#pragma unroll
      for (int j = 0; j < NSRC; ++j) {
        float g[8];
        unpack8(raw[j], g);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          a.x[k] = (j == 0) ? acc_op<MODE>(a.x[k], g[k], w) : fmaf(w, g[k], a.x[k]);
      }
      if (wide) {
        st8(dst + e, a);
      } else {
        *reinterpret_cast<float4*>(dst + e) = make_float4(a.x[0], a.x[1], a.x[2], a.x[3]);
        *reinterpret_cast<float4*>(dst + e + 4) = make_float4(a.x[4], a.x[5], a.x[6], a.x[7]);
      }
    } else {
      const int64_t end = base + kChunk < sg.n ? base + kChunk : sg.n;
      for (int64_t e = base + threadIdx.x; e < end; e += 512) {
        float a = acc_op<MODE>((MODE & HET_ACC_FIRST) ? 0.f : dst[e],
                               __bfloat162float(src[0][e]), w);
#pragma unroll
        for (int j = 1; j < NSRC; ++j) a = fmaf(w, __bfloat162float(src[j][e]), a);
        dst[e] = a;
      }
    }
  }
}

// bf16 segments copied into one bf16 buffer (persistent grid, as accumulate);
// a CTA chunk is 512 threads x 2 x 16 B, both loads issued before the stores
constexpr int kGatherIters = 2;
constexpr int64_t kGatherChunk = 512 * 8 * kGatherIters;

__global__ void __launch_bounds__(512) gather_bf16_kernel(__nv_bfloat16* __restrict__ dst,
                                                          const __grid_constant__ SegTable t) {
  const int64_t total = t.first_block[t.nseg];
  int64_t b = blockIdx.x;
  if (b >= total) return;
  int lo = 0, hi = t.nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (t.first_block[mid] <= b) lo = mid; else hi = mid - 1;
  }
  int s = lo;
  for (; b < total; b += gridDim.x) {
    while (s + 1 < t.nseg && t.first_block[s + 1] <= b) ++s;
    const het_seg_t sg = t.seg[s];
    const int64_t base = (b - t.first_block[s]) * kGatherChunk;
    const __nv_bfloat16* src = static_cast<const __nv_bfloat16*>(sg.src);
    __nv_bfloat16* d = dst + sg.dst_off;
    const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(d)) & 15) == 0;
    if (vec && base + kGatherChunk <= sg.n) {
      uint4 r[kGatherIters];
#pragma unroll
      for (int it = 0; it < kGatherIters; ++it)
        r[it] = __ldcs(reinterpret_cast<const uint4*>(src + base + (it * 512 + threadIdx.x) * 8));
#pragma unroll
      for (int it = 0; it < kGatherIters; ++it)
        *reinterpret_cast<uint4*>(d + base + (it * 512 + threadIdx.x) * 8) = r[it];
    } else {
      const int64_t end = base + kGatherChunk < sg.n ? base + kGatherChunk : sg.n;
      for (int64_t i = base + threadIdx.x; i < end; i += 512) d[i] = src[i];
    }
  }
}

// ---------------------------------------------------------------- AdamW

struct AdamCoef {
  float decay;        // 1 - lr * wd
  float one_m_b1;     // 1 - beta1
  float beta2;
  float one_m_b2;     // 1 - beta2
  float bc2_sqrt;  // sqrt(1 - beta2^t)  (divisor, as torch)
  float eps;
  float neg_step;     // -lr / (1 - beta1^t)
};

// Rounding is pinned with explicit intrinsics (no compiler contraction), so
// the oracle (oracle/step_oracle.adamw) can mirror it operation for operation.
__device__ __forceinline__ void adam1(float& p, float g, float& m, float& v, const AdamCoef& c) {
  p = __fmul_rn(p, c.decay);                                  // p *= 1 - lr*wd
  m = __fmaf_rn(c.one_m_b1, __fsub_rn(g, m), m);              // m.lerp_(g, 1 - b1)
  v = __fmaf_rn(__fmul_rn(c.one_m_b2, g), g, __fmul_rn(v, c.beta2));  // v*b2 + (1-b2) g^2
  const float denom = __fadd_rn(__fdiv_rn(__fsqrt_rn(v), c.bc2_sqrt), c.eps);
  p = __fmaf_rn(c.neg_step, __fdiv_rn(m, denom), p);          // p.addcdiv_(m, denom, -lr/bc1)
}

template <bool SHADOW>
__global__ void __launch_bounds__(kThreads) adamw_vec_kernel(float4* __restrict__ p,
                                                             const float4* __restrict__ g,
                                                             float4* __restrict__ m,
                                                             float4* __restrict__ v,
                                                             uint2* __restrict__ shadow,
                                                             int64_t n4, AdamCoef c,
                                                             const AdamCoef* __restrict__ cdev) {
  if (cdev != nullptr) c = *cdev;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += 2 * stride) {
    const int64_t j = i + stride;
    const bool two = j < n4;
    float4 p0 = p[i], g0 = __ldcs(g + i), m0 = m[i], v0 = v[i];
    float4 p1, g1, m1, v1;
    if (two) {
      p1 = p[j];
      g1 = __ldcs(g + j);
      m1 = m[j];
      v1 = v[j];
    }
    adam1(p0.x, g0.x, m0.x, v0.x, c);
    adam1(p0.y, g0.y, m0.y, v0.y, c);
    adam1(p0.z, g0.z, m0.z, v0.z, c);
    adam1(p0.w, g0.w, m0.w, v0.w, c);
    p[i] = p0;
    m[i] = m0;
    v[i] = v0;
    if (SHADOW) shadow[i] = make_uint2(pack2(p0.x, p0.y), pack2(p0.z, p0.w));
    if (two) {
      adam1(p1.x, g1.x, m1.x, v1.x, c);
      adam1(p1.y, g1.y, m1.y, v1.y, c);
      adam1(p1.z, g1.z, m1.z, v1.z, c);
      adam1(p1.w, g1.w, m1.w, v1.w, c);
      p[j] = p1;
      m[j] = m1;
      v[j] = v1;
      if (SHADOW) shadow[j] = make_uint2(pack2(p1.x, p1.y), pack2(p1.z, p1.w));
    }
  }
}

// 256-bit variant: 8 params per thread per iteration (32 B of each state
// stream), shadow as one 16-byte store. Used when every stream is 32B-aligned.
template <bool SHADOW>
__global__ void __launch_bounds__(kThreads) adamw_v8_kernel(float* __restrict__ p,
                                                            const float* __restrict__ g,
                                                            float* __restrict__ m,
                                                            float* __restrict__ v,
                                                            uint4* __restrict__ shadow,
                                                            int64_t n8, AdamCoef c,
                                                            const AdamCoef* __restrict__ cdev) {
  if (cdev != nullptr) c = *cdev;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n8;
       i += stride) {
    F8 P = ld8(p + i * 8), G = ld8_stream(g + i * 8), M = ld8(m + i * 8), V = ld8(v + i * 8);
#pragma unroll
    for (int k = 0; k < 8; ++k) adam1(P.x[k], G.x[k], M.x[k], V.x[k], c);
    st8(p + i * 8, P);
    st8(m + i * 8, M);
    st8(v + i * 8, V);
    if (SHADOW)
      shadow[i] = make_uint4(pack2(P.x[0], P.x[1]), pack2(P.x[2], P.x[3]), pack2(P.x[4], P.x[5]),
                             pack2(P.x[6], P.x[7]));
  }
}

__global__ void adamw_scalar_kernel(float* __restrict__ p, const float* __restrict__ g,
                                    float* __restrict__ m, float* __restrict__ v,
                                    __nv_bfloat16* __restrict__ shadow, int64_t n, AdamCoef c,
                                    const AdamCoef* __restrict__ cdev) {
  if (cdev != nullptr) c = *cdev;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride) {
    float pp = p[i], mm = m[i], vv = v[i];
    adam1(pp, g[i], mm, vv, c);
    p[i] = pp;
    m[i] = mm;
    v[i] = vv;
    if (shadow) shadow[i] = __float2bfloat16_rn(pp);
  }
}

// ---------------------------------------------------------------- embedding grad

// blockIdx.x < nseg: token run; otherwise position row (wpe). Each thread owns
// kVecE columns of the row (d <= kThreads * kVecE).
constexpr int kVecE = 8;

__global__ void __launch_bounds__(kThreads) embedding_grad_kernel(
    float* __restrict__ acc, int64_t wte_off, int64_t wpe_off,
    const __nv_bfloat16* __restrict__ dy, int64_t rows, int64_t d,
    const int32_t* __restrict__ order, const int32_t* __restrict__ seg_start,
    const int32_t* __restrict__ seg_token, int64_t nseg, int64_t seq, float w,
    const int32_t* __restrict__ nseg_dev) {
  int64_t b = blockIdx.x;
  if (nseg_dev != nullptr) {
    // device-side run count: blocks [0, nseg) are token runs (nseg = the host's
    // upper bound on runs), blocks past the live count exit; seg_token is the
    // sorted token array, read at each run's start
    if (b < nseg) {
      if (b >= *nseg_dev) return;
    }
  }
  for (int64_t c0 = static_cast<int64_t>(threadIdx.x) * kVecE; c0 < d;
       c0 += static_cast<int64_t>(blockDim.x) * kVecE) {
    float sum[kVecE];
#pragma unroll
    for (int k = 0; k < kVecE; ++k) sum[k] = 0.f;
    const bool vec = c0 + kVecE <= d && (d % kVecE) == 0;
    auto add_row = [&](int64_t r) {
      const __nv_bfloat16* row = dy + r * d + c0;
      if (vec) {
        float f[8];
        unpack8(*reinterpret_cast<const uint4*>(row), f);
#pragma unroll
        for (int k = 0; k < kVecE; ++k) sum[k] += f[k];
      } else {
        for (int k = 0; k < kVecE && c0 + k < d; ++k) sum[k] += __bfloat162float(row[k]);
      }
    };
    int64_t dst;
    if (b < nseg) {
      for (int32_t i = seg_start[b]; i < seg_start[b + 1]; ++i) add_row(order[i]);
      const int32_t tok = nseg_dev != nullptr ? seg_token[seg_start[b]] : seg_token[b];
      dst = wte_off + static_cast<int64_t>(tok) * d + c0;
    } else {
      const int64_t s = b - nseg;
      for (int64_t r = s; r < rows; r += seq) add_row(r);
      dst = wpe_off + s * d + c0;
    }
    for (int k = 0; k < kVecE && c0 + k < d; ++k) acc[dst + k] = fmaf(w, sum[k], acc[dst + k]);
  }
}

__global__ void fill_kernel(float* __restrict__ dst, float value, int64_t n) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += stride)
    dst[i] = value;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

namespace {
// Diagnostic for the heterogeneity emulation: each CTA records the SM it ran
// on (%smid), so a test can prove a green-context stream stays in its partition.
__global__ void probe_smid_kernel(int32_t* out) {
  if (threadIdx.x == 0) {
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    // keep the CTA resident a little so the launch spreads over the partition
    const long long t0 = clock64();
    while (clock64() - t0 < 20000) {
    }
    out[blockIdx.x] = static_cast<int32_t>(sm);
  }
}

}  // namespace

extern "C" {

const char* het_version(void) { return "hetstep 0.1.0 sm_100a"; }

const char* het_last_error(void) { return het::g_last_error.c_str(); }

int het_pack_bf16(const float* src, void* dst_bf16, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!src || !dst_bf16))) return fail(HET_EARG, "het_pack_bf16: bad args");
  if (n == 0) return HET_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (aligned16(src) && (reinterpret_cast<uintptr_t>(dst_bf16) & 7) == 0 && n % 4 == 0) {
    const int64_t n4 = n / 4;
    pack_vec_kernel<<<het::grid_for((n4 + 1) / 2, kThreads), kThreads, 0, st>>>(
        reinterpret_cast<const float4*>(src), static_cast<uint2*>(dst_bf16), n4);
  } else {
    pack_scalar_kernel<<<het::grid_for(n, kThreads), kThreads, 0, st>>>(
        src, static_cast<__nv_bfloat16*>(dst_bf16), n);
  }
  return het::check_launch("het_pack_bf16");
}

int het_accumulate(float* acc, const het_seg_t* segs, int nseg, int mode, float scale,
                   void* stream) {
  if (!acc || !segs || nseg < 1 || nseg > HET_MAX_SEGS || (mode != HET_ACC_ADD && mode != HET_ACC_FIRST))
    return fail(HET_EARG, "het_accumulate: bad args (nseg=%d mode=%d)", nseg, mode);
  SegTable t;
  t.nseg = nseg;
  const AccShape shape = kAccShapes[g_acc_variant];
  const int64_t chunk = static_cast<int64_t>(shape.threads) * kAccVec * shape.iters;
  int64_t blocks = 0;
  for (int s = 0; s < nseg; ++s) {
    if (segs[s].n < 0 || segs[s].dst_off < 0 || (segs[s].n > 0 && !segs[s].src))
      return fail(HET_EARG, "het_accumulate: bad segment %d", s);
    t.seg[s] = segs[s];
    t.first_block[s] = blocks;
    blocks += (segs[s].n + chunk - 1) / chunk;
  }
  t.first_block[nseg] = blocks;
  for (int s = nseg + 1; s <= HET_MAX_SEGS; ++s) t.first_block[s] = blocks;
  if (blocks == 0) return HET_OK;
  if (blocks > 0x7fffffff) return fail(HET_EARG, "het_accumulate: too large");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // persistent: at most the resident CTAs of the variant (occupancy per SM cached per
  // variant) on the SMs this rank may use (green-context budget, het::sm_count)
  static int resident[8][2] = {};
#define HET_ACC_LAUNCH(T, I)                                                              \
  do {                                                                                    \
    auto kf = mode == HET_ACC_FIRST ? accumulate_kernel<HET_ACC_FIRST, T, I>              \
                                    : accumulate_kernel<HET_ACC_ADD, T, I>;               \
    int& per_sm = resident[g_acc_variant][mode == HET_ACC_FIRST];                         \
    if (per_sm == 0) {                                                                    \
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf, T, 0);                   \
      if (per_sm <= 0) per_sm = 1;                                                        \
    }                                                                                     \
    const int64_t r = het::g_acc_grid ? blocks : static_cast<int64_t>(per_sm) *          \
                                                 het::sm_count();                         \
    const dim3 grid(static_cast<unsigned>(blocks < r ? blocks : r));                      \
    kf<<<grid, T, 0, st>>>(acc, t, scale);                                                \
  } while (0)
  switch (g_acc_variant) {
    case 1: HET_ACC_LAUNCH(256, 2); break;
    case 2: HET_ACC_LAUNCH(256, 1); break;
    case 3: HET_ACC_LAUNCH(512, 2); break;
    case 4: HET_ACC_LAUNCH(512, 1); break;
    case 5: HET_ACC_LAUNCH(128, 4); break;
    default: HET_ACC_LAUNCH(256, 4);
  }
#undef HET_ACC_LAUNCH
  return het::check_launch("het_accumulate");
}

int het_accumulate_multi(float* acc, const het_seg_t* segs, int nseg, int nsrc, int mode,
                         float scale, void* stream) {
  if (!acc || !segs || nseg < 1 || nseg > HET_MAX_SEGS || nsrc < 1 || nsrc > HET_MAX_ACC_SRC ||
      (mode != HET_ACC_ADD && mode != HET_ACC_FIRST))
    return fail(HET_EARG, "het_accumulate_multi: bad args (nseg=%d nsrc=%d mode=%d)", nseg,
                nsrc, mode);
  SegTable t;
  MoreSrc ms;
  std::memset(&ms, 0, sizeof(ms));
  t.nseg = nseg;
  constexpr int64_t chunk = 512 * kAccVec;
  int64_t blocks = 0;
  for (int s = 0; s < nseg; ++s) {
    const het_seg_t& s0 = segs[s];
    if (s0.n < 0 || s0.dst_off < 0 || (s0.n > 0 && !s0.src))
      return fail(HET_EARG, "het_accumulate_multi: bad segment %d", s);
    for (int j = 1; j < nsrc; ++j) {
      const het_seg_t& sj = segs[static_cast<int64_t>(j) * nseg + s];
      if (sj.n != s0.n || sj.dst_off != s0.dst_off || (s0.n > 0 && !sj.src))
        return fail(HET_EARG, "het_accumulate_multi: source %d of segment %d differs in shape",
                    j, s);
      ms.src[j - 1][s] = sj.src;
    }
    t.seg[s] = s0;
    t.first_block[s] = blocks;
    blocks += (s0.n + chunk - 1) / chunk;
  }
  for (int s = nseg; s <= HET_MAX_SEGS; ++s) t.first_block[s] = blocks;
  if (blocks == 0) return HET_OK;
  if (blocks > 0x7fffffff) return fail(HET_EARG, "het_accumulate_multi: too large");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm,
                                                  accumulate_multi_kernel<HET_ACC_ADD, 4>, 512, 0);
    if (per_sm <= 0) per_sm = 1;
  }
  const int64_t resident = het::g_acc_grid ? blocks
                                           : static_cast<int64_t>(per_sm) * het::sm_count();
  const dim3 grid(static_cast<unsigned>(blocks < resident ? blocks : resident));
#define HET_ACCM(M, K) accumulate_multi_kernel<M, K><<<grid, 512, 0, st>>>(acc, t, ms, scale)
  if (mode == HET_ACC_FIRST) {
    switch (nsrc) {
      case 1: HET_ACCM(HET_ACC_FIRST, 1); break;
      case 2: HET_ACCM(HET_ACC_FIRST, 2); break;
      case 3: HET_ACCM(HET_ACC_FIRST, 3); break;
      default: HET_ACCM(HET_ACC_FIRST, 4);
    }
  } else {
    switch (nsrc) {
      case 1: HET_ACCM(HET_ACC_ADD, 1); break;
      case 2: HET_ACCM(HET_ACC_ADD, 2); break;
      case 3: HET_ACCM(HET_ACC_ADD, 3); break;
      default: HET_ACCM(HET_ACC_ADD, 4);
    }
  }
#undef HET_ACCM
  return het::check_launch("het_accumulate_multi");
}

int het_gather_bf16(void* dst, const het_seg_t* segs, int nseg, void* stream) {
  if (!dst || !segs || nseg < 1 || nseg > HET_MAX_SEGS)
    return fail(HET_EARG, "het_gather_bf16: bad args (nseg=%d)", nseg);
  SegTable t;
  t.nseg = nseg;
  int64_t blocks = 0;
  for (int s = 0; s < nseg; ++s) {
    if (segs[s].n < 0 || segs[s].dst_off < 0 || (segs[s].n > 0 && !segs[s].src))
      return fail(HET_EARG, "het_gather_bf16: bad segment %d", s);
    t.seg[s] = segs[s];
    t.first_block[s] = blocks;
    blocks += (segs[s].n + kGatherChunk - 1) / kGatherChunk;
  }
  for (int s = nseg; s <= HET_MAX_SEGS; ++s) t.first_block[s] = blocks;
  if (blocks == 0) return HET_OK;
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gather_bf16_kernel, 512, 0);
    if (per_sm <= 0) per_sm = 1;
  }
  const int64_t resident = static_cast<int64_t>(per_sm) * het::sm_count();
  const unsigned grid = static_cast<unsigned>(blocks < resident ? blocks : resident);
  gather_bf16_kernel<<<grid, 512, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<__nv_bfloat16*>(dst), t);
  return het::check_launch("het_gather_bf16");
}

int het_adamw_coef(double lr, double beta1, double beta2, double eps, double weight_decay,
                   int64_t step, float* out7) {
  if (step < 1 || !out7) return fail(HET_EARG, "het_adamw_coef: bad args (step=%lld)",
                                     (long long)step);
  // scalar coefficients in double, as torch's _single_tensor_adamw computes them
  const double bc1 = 1.0 - std::pow(beta1, static_cast<double>(step));
  const double bc2 = 1.0 - std::pow(beta2, static_cast<double>(step));
  AdamCoef c;
  c.decay = static_cast<float>(1.0 - lr * weight_decay);
  c.one_m_b1 = static_cast<float>(1.0 - beta1);
  c.beta2 = static_cast<float>(beta2);
  c.one_m_b2 = static_cast<float>(1.0 - beta2);
  c.bc2_sqrt = static_cast<float>(std::sqrt(bc2));
  c.eps = static_cast<float>(eps);
  c.neg_step = static_cast<float>(-(lr / bc1));
  static_assert(sizeof(AdamCoef) == 7 * sizeof(float), "AdamCoef layout");
  std::memcpy(out7, &c, sizeof(c));
  return HET_OK;
}

namespace {

int adamw_launch(float* p, const float* g, float* m, float* v, void* p_bf16_or_null, int64_t n,
                 const AdamCoef& c, const AdamCoef* cdev, void* stream, const char* what) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool wide = n % 8 == 0 && aligned32(p) && aligned32(g) && aligned32(m) && aligned32(v) &&
                    (!p_bf16_or_null || aligned16(p_bf16_or_null));
  const bool vec = n % 4 == 0 && aligned16(p) && aligned16(g) && aligned16(m) && aligned16(v) &&
                   (!p_bf16_or_null || (reinterpret_cast<uintptr_t>(p_bf16_or_null) & 7) == 0);
  if (wide) {
    const int64_t n8 = n / 8;
    const int grid = het::grid_for(n8, kThreads);
    if (p_bf16_or_null)
      adamw_v8_kernel<true><<<grid, kThreads, 0, st>>>(
          p, g, m, v, static_cast<uint4*>(p_bf16_or_null), n8, c, cdev);
    else
      adamw_v8_kernel<false><<<grid, kThreads, 0, st>>>(p, g, m, v, nullptr, n8, c, cdev);
  } else if (vec) {
    const int64_t n4 = n / 4;
    const int grid = het::grid_for((n4 + 1) / 2, kThreads);
    if (p_bf16_or_null)
      adamw_vec_kernel<true><<<grid, kThreads, 0, st>>>(
          reinterpret_cast<float4*>(p), reinterpret_cast<const float4*>(g),
          reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v),
          static_cast<uint2*>(p_bf16_or_null), n4, c, cdev);
    else
      adamw_vec_kernel<false><<<grid, kThreads, 0, st>>>(
          reinterpret_cast<float4*>(p), reinterpret_cast<const float4*>(g),
          reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), nullptr, n4, c, cdev);
  } else {
    adamw_scalar_kernel<<<het::grid_for(n, kThreads), kThreads, 0, st>>>(
        p, g, m, v, static_cast<__nv_bfloat16*>(p_bf16_or_null), n, c, cdev);
  }
  return het::check_launch(what);
}

}  // namespace

int het_adamw(float* p, const float* g, float* m, float* v, void* p_bf16_or_null, int64_t n,
              double lr, double beta1, double beta2, double eps, double weight_decay,
              int64_t step, void* stream) {
  if (n < 0 || step < 1 || (n > 0 && (!p || !g || !m || !v)))
    return fail(HET_EARG, "het_adamw: bad args (n=%lld step=%lld)", (long long)n,
                (long long)step);
  if (n == 0) return HET_OK;
  AdamCoef c;
  het_adamw_coef(lr, beta1, beta2, eps, weight_decay, step, reinterpret_cast<float*>(&c));
  return adamw_launch(p, g, m, v, p_bf16_or_null, n, c, nullptr, stream, "het_adamw");
}

int het_adamw_devcoef(float* p, const float* g, float* m, float* v, void* p_bf16_or_null,
                      int64_t n, const float* coef7_dev, void* stream) {
  if (n < 0 || !coef7_dev || (n > 0 && (!p || !g || !m || !v)))
    return fail(HET_EARG, "het_adamw_devcoef: bad args (n=%lld)", (long long)n);
  if (n == 0) return HET_OK;
  AdamCoef unused{};
  return adamw_launch(p, g, m, v, p_bf16_or_null, n, unused,
                      reinterpret_cast<const AdamCoef*>(coef7_dev), stream, "het_adamw_devcoef");
}

int het_embedding_grad(float* acc, int64_t wte_off, int64_t wpe_off, const void* dy_bf16,
                       int64_t rows, int64_t d, const int32_t* order, const int32_t* seg_start,
                       const int32_t* seg_token, int64_t nseg, int64_t seq, float scale,
                       void* stream) {
  if (!acc || !dy_bf16 || rows < 0 || d <= 0 || nseg < 0 || seq <= 0 || wte_off < 0 ||
      (nseg > 0 && (!order || !seg_start || !seg_token)))
    return fail(HET_EARG, "het_embedding_grad: bad args");
  const int64_t blocks = nseg + (wpe_off >= 0 ? seq : 0);
  if (blocks == 0 || rows == 0) return HET_OK;
  embedding_grad_kernel<<<static_cast<unsigned>(blocks), kThreads, 0,
                          static_cast<cudaStream_t>(stream)>>>(
      acc, wte_off, wpe_off, static_cast<const __nv_bfloat16*>(dy_bf16), rows, d, order,
      seg_start, seg_token, nseg, seq, scale, nullptr);
  return het::check_launch("het_embedding_grad");
}

int het_embedding_grad_dev(float* acc, int64_t wte_off, int64_t wpe_off, const void* dy_bf16,
                           int64_t rows, int64_t d, const int32_t* order,
                           const int32_t* seg_start, const int32_t* sorted_tok,
                           const int32_t* nseg_dev, int64_t seq, float scale, void* stream) {
  if (!acc || !dy_bf16 || rows < 0 || d <= 0 || seq <= 0 || wte_off < 0 ||
      (rows > 0 && (!order || !seg_start || !sorted_tok || !nseg_dev)))
    return fail(HET_EARG, "het_embedding_grad_dev: bad args");
  if (rows == 0) return HET_OK;
  const int64_t blocks = rows + (wpe_off >= 0 ? seq : 0);   // rows bounds the token runs
  embedding_grad_kernel<<<static_cast<unsigned>(blocks), kThreads, 0,
                          static_cast<cudaStream_t>(stream)>>>(
      acc, wte_off, wpe_off, static_cast<const __nv_bfloat16*>(dy_bf16), rows, d, order,
      seg_start, sorted_tok, rows, seq, scale, nseg_dev);
  return het::check_launch("het_embedding_grad_dev");
}

int het_tune(int key, int value) {
  if (key == HET_TUNE_SM_BUDGET) {
    if (value < 0) return fail(HET_EARG, "het_tune: SM budget must be >= 0");
    het::g_sm_budget = value;
    return HET_OK;
  }
  if (key == HET_TUNE_SYMM_TIMEOUT_MS) return het::set_symm_timeout_ms(value);
  if (key == HET_TUNE_ACC_GRID) {
    if (value != 0 && value != 1) return fail(HET_EARG, "het_tune: accumulate grid mode 0 or 1");
    het::g_acc_grid = value;
    return HET_OK;
  }
  if (key == HET_TUNE_ACC_VARIANT) {
    if (value < 0 || value >= static_cast<int>(sizeof(kAccShapes) / sizeof(kAccShapes[0])))
      return fail(HET_EARG, "het_tune: accumulate variant %d out of range", value);
    g_acc_variant = value;
    return HET_OK;
  }
  return fail(HET_EARG, "het_tune: unknown key %d", key);
}

int het_probe_smid(int32_t* out, int ctas, void* stream) {
  if (!out || ctas < 1) return fail(HET_EARG, "het_probe_smid: bad args");
  probe_smid_kernel<<<ctas, 128, 0, static_cast<cudaStream_t>(stream)>>>(out);
  return het::check_launch("het_probe_smid");
}

int het_fill_f32(float* dst, float value, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && !dst)) return fail(HET_EARG, "het_fill_f32: bad args");
  if (n == 0) return HET_OK;
  fill_kernel<<<het::grid_for(n, kThreads), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      dst, value, n);
  return het::check_launch("het_fill_f32");
}

}  // extern "C"

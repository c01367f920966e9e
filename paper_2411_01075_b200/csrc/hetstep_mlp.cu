// Model-side linear-layer epilogues for the GPT/BERT units (bf16 in/out,
// fp32 sums): the bias gradient as a deterministic column sum, and the tanh
// GELU forward / backward, the backward fused with the bias gradient of the
// layer that produced GELU's input. Not owned hot-path rows, but the largest
// non-GEMM costs left in the unit (torch's bias-grad reduction runs at ~2.3
// TB/s, GELU backward and the reduction re-read the same [rows, n] tensor).
//
// Column sums: a CTA of 32 x 8 threads owns 32*V columns and one chunk of
// rows; lane x sums its V columns over the rows y, y+8, ... of the chunk, the
// 8 row lanes meet in shared memory and the CTA writes one fp32 partial row.
// A finalize pass sums the partial rows in fixed order (deterministic).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "hetstep.h"
#include "hetstep_internal.cuh"

using het::fail;

namespace {

constexpr int kRowLanes = 8;
constexpr int kTargetCtas = 148 * 4;

__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 raw = __ldcs(reinterpret_cast<const uint4*>(p));
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float((w[i] & 0xffffu) << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

// round to bf16 and back (the value torch's bf16 tensors hold)
__device__ __forceinline__ float rbf(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// torch's tanh-approximate GELU, y = 0.5 x (1 + tanh(u)), u = b (x + k x^3),
// and its derivative, evaluated through 0.5 (1 + tanh(u)) = sigmoid(2u):
//   y = x s,  dy/dx = s + x s (1 - s) 2u' = s (1 + x e s (c0 + 3 c1 x^2)),
//   s = 1 / (1 + e), e = exp(-2u), 2u = x (c0 + c1 x^2), c0 = 2b, c1 = 2bk.
// One ex2 and one rcp (MUFU) and about ten FP32 instructions per element, no
// cancellation (1 + tanh(u) is never formed), against torch's tanhf form at
// about twenty (both kernels were issue-bound on it: 78% issue slots busy at
// 0.65 of HBM in ncu). Agrees with torch's fp32 formula to a few fp32 ulps;
// after bf16 rounding the outputs match torch's except for rare 1-ulp ties
// (tests/test_kernels_gpu.py bounds both).
constexpr float kC0 = 1.5957691216057308f;          // 2 sqrt(2/pi)
constexpr float kC1 = 0.07135481627159701f;         // 2 sqrt(2/pi) 0.044715
constexpr float kNegLog2e = -1.4426950408889634f;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// e = exp(-2u), clamped at 2^80 so that e * s stays finite for very negative x
__device__ __forceinline__ float gelu_e(float x, float x_sq) {
  const float t = x * fmaf(kC1 * kNegLog2e, x_sq, kC0 * kNegLog2e);
  return ex2_approx(fminf(t, 80.f));
}

__device__ __forceinline__ float gelu_f(float x) {
  const float e = gelu_e(x, x * x);
  return x * rcp_approx(1.f + e);
}

__device__ __forceinline__ float gelu_grad_f(float dy, float x) {
  const float x_sq = x * x;
  const float e = gelu_e(x, x_sq);
  const float s = rcp_approx(1.f + e);
  const float du = fmaf(3.f * kC1, x_sq, kC0);
  return dy * (s * fmaf(x * e * s, du, 1.f));
}

// What a column-sum pass sums, per element: the bias gradient sums g itself;
// the GELU backward writes dpre = GELU'(pre) * g and sums the rounded dpre.
struct BiasOnly {
  const __nv_bfloat16* g;
  template <int V>
  __device__ __forceinline__ void row(int64_t off, float (&v)[V]) const {
    if constexpr (V == 8) {
      ld8(g + off, v);
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = __bfloat162float(g[off + i]);
    }
  }
};

struct GeluBwd {
  const __nv_bfloat16* g;
  const __nv_bfloat16* pre;
  __nv_bfloat16* dpre;
  template <int V>
  __device__ __forceinline__ void row(int64_t off, float (&v)[V]) const {
    float gv[V], xv[V];
    if constexpr (V == 8) {
      ld8(g + off, gv);
      ld8(pre + off, xv);
    } else {
#pragma unroll
      for (int i = 0; i < V; ++i) {
        gv[i] = __bfloat162float(g[off + i]);
        xv[i] = __bfloat162float(pre[off + i]);
      }
    }
    __nv_bfloat16 o[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      o[i] = __float2bfloat16_rn(gelu_grad_f(gv[i], xv[i]));
      v[i] = __bfloat162float(o[i]);
    }
    if constexpr (V == 8)
      *reinterpret_cast<uint4*>(dpre + off) = *reinterpret_cast<const uint4*>(o);
    else
#pragma unroll
      for (int i = 0; i < V; ++i) dpre[off + i] = o[i];
  }
};

// 4 CTAs per SM (<= 64 registers): plan_colsum sizes the grid to one full
// wave of 148 * 4 CTAs; at 3 resident CTAs (75 registers, the GELU backward
// before the bound) the same grid ran 1.3 waves
template <class Op, int V>
__global__ void __launch_bounds__(32 * kRowLanes, 4) colsum_kernel(Op op, int64_t rows, int64_t n,
                                                                int64_t chunk_rows,
                                                                float* __restrict__ partial) {
  __shared__ float red[kRowLanes][32 * V];
  const int64_t col = (static_cast<int64_t>(blockIdx.x) * 32 + threadIdx.x) * V;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * chunk_rows;
  const int64_t r1 = r0 + chunk_rows < rows ? r0 + chunk_rows : rows;
  float acc[V];
#pragma unroll
  for (int i = 0; i < V; ++i) acc[i] = 0.f;
  if (col < n) {
    constexpr int kRows = 4;                   // rows in flight per thread
    for (int64_t r = r0 + threadIdx.y; r < r1; r += kRows * kRowLanes) {
      float v[kRows][V];
#pragma unroll
      for (int j = 0; j < kRows; ++j) {
        if (r + j * kRowLanes < r1) {
          op.template row<V>((r + j * kRowLanes) * n + col, v[j]);
        } else {
#pragma unroll
          for (int i = 0; i < V; ++i) v[j][i] = 0.f;
        }
      }
#pragma unroll
      for (int j = 0; j < kRows; ++j)
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] += v[j][i];
    }
  }
#pragma unroll
  for (int i = 0; i < V; ++i) red[threadIdx.y][threadIdx.x * V + i] = acc[i];
  __syncthreads();
  // the CTA's 32*V columns, summed over the 8 row lanes in fixed order
  for (int c = threadIdx.y * 32 + threadIdx.x; c < 32 * V; c += 32 * kRowLanes) {
    float t = 0.f;
#pragma unroll
    for (int y = 0; y < kRowLanes; ++y) t += red[y][c];
    const int64_t gc = static_cast<int64_t>(blockIdx.x) * 32 * V + c;
    if (gc < n) partial[static_cast<int64_t>(blockIdx.y) * n + gc] = t;
  }
}

// db[c] = bf16(sum over chunks of partial[k][c]), 32 columns per CTA, 8 warps over
// chunks with 8 independent sums each (loads in flight; fixed order)
__global__ void __launch_bounds__(256) colsum_finalize_kernel(const float* __restrict__ partial,
                                                              int chunks, int64_t n,
                                                              __nv_bfloat16* __restrict__ db) {
  __shared__ float red[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * 32 + lane;
  float acc = 0.f;
  if (c < n) {
    float p8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int k = warp;
    for (; k + 56 < chunks; k += 64) {
#pragma unroll
      for (int j = 0; j < 8; ++j) p8[j] += partial[static_cast<int64_t>(k + 8 * j) * n + c];
    }
    for (; k < chunks; k += 8) p8[0] += partial[static_cast<int64_t>(k) * n + c];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += p8[j];
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && c < n) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][lane];
    db[c] = __float2bfloat16_rn(t);
  }
}

// grid-stride; the vector form keeps two 16-byte loads in flight per thread
template <int V>
__global__ void gelu_fwd_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                int64_t n) {
  const int64_t items = n / V;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if constexpr (V == 8) {
    for (; t < items; t += 2 * stride) {
      const bool two = t + stride < items;
      float f[2][8];
      ld8(x + t * 8, f[0]);
      if (two) ld8(x + (t + stride) * 8, f[1]);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (k == 1 && !two) break;
        __nv_bfloat16 o[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = __float2bfloat16_rn(gelu_f(f[k][i]));
        *reinterpret_cast<uint4*>(y + (t + k * stride) * 8) = *reinterpret_cast<const uint4*>(o);
      }
    }
  } else {
    for (; t < items; t += stride) y[t] = __float2bfloat16_rn(gelu_f(__bfloat162float(x[t])));
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

struct Plan {
  int v;
  unsigned col_tiles;
  int chunks;
  int64_t chunk_rows;
};

Plan plan_colsum(int64_t rows, int64_t n, bool vec) {
  Plan p;
  p.v = vec ? 8 : 1;
  p.col_tiles = static_cast<unsigned>((n + 32 * p.v - 1) / (32 * p.v));
  int64_t chunks = kTargetCtas / static_cast<int64_t>(p.col_tiles);
  if (chunks < 1) chunks = 1;
  const int64_t min_rows = 4 * kRowLanes;      // at least 4 rows per row lane
  if (chunks > (rows + min_rows - 1) / min_rows) chunks = (rows + min_rows - 1) / min_rows;
  if (chunks < 1) chunks = 1;
  p.chunk_rows = (rows + chunks - 1) / chunks;
  p.chunks = static_cast<int>((rows + p.chunk_rows - 1) / p.chunk_rows);
  if (p.chunks < 1) p.chunks = 1;
  return p;
}

template <class Op>
int run_colsum(const Op& op, bool vec, int64_t rows, int64_t n, void* db, float* partial,
               void* stream, const char* what) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Plan p = plan_colsum(rows, n, vec);
  const dim3 grid(p.col_tiles, static_cast<unsigned>(p.chunks)), block(32, kRowLanes);
  if (p.v == 8)
    colsum_kernel<Op, 8><<<grid, block, 0, st>>>(op, rows, n, p.chunk_rows, partial);
  else
    colsum_kernel<Op, 1><<<grid, block, 0, st>>>(op, rows, n, p.chunk_rows, partial);
  int rc = het::check_launch(what);
  if (rc != HET_OK) return rc;
  colsum_finalize_kernel<<<static_cast<unsigned>((n + 31) / 32), 256, 0, st>>>(
      partial, p.chunks, n, static_cast<__nv_bfloat16*>(db));
  return het::check_launch(what);
}

}  // namespace

extern "C" {

int64_t het_colsum_partial_floats(int64_t rows, int64_t n) {
  if (rows <= 0 || n <= 0) return 1;
  const Plan p = plan_colsum(rows, n, n % 8 == 0);
  return static_cast<int64_t>(p.chunks) * n;
}

int het_bias_grad(const void* g, int64_t rows, int64_t n, void* db, float* partial, void* stream) {
  if (!g || !db || !partial || rows < 0 || n <= 0) return fail(HET_EARG, "het_bias_grad: bad args");
  if (rows == 0) {
    return cudaMemsetAsync(db, 0, n * 2, static_cast<cudaStream_t>(stream)) == cudaSuccess
               ? HET_OK
               : fail(HET_ECUDA, "het_bias_grad: memset failed");
  }
  const bool vec = n % 8 == 0 && aligned16(g);
  return run_colsum(BiasOnly{static_cast<const __nv_bfloat16*>(g)}, vec, rows, n, db, partial,
                    stream, "het_bias_grad");
}

int het_gelu_fwd(const void* x, void* y, int64_t n, void* stream) {
  if (!x || !y || n < 0) return fail(HET_EARG, "het_gelu_fwd: bad args");
  if (n == 0) return HET_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool vec = n % 8 == 0 && aligned16(x) && aligned16(y);
  const int64_t items = vec ? n / 8 : n;
  int64_t blocks = (items + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  auto X = static_cast<const __nv_bfloat16*>(x);
  auto Y = static_cast<__nv_bfloat16*>(y);
  if (vec)
    gelu_fwd_kernel<8><<<static_cast<unsigned>(blocks), 256, 0, st>>>(X, Y, n);
  else
    gelu_fwd_kernel<1><<<static_cast<unsigned>(blocks), 256, 0, st>>>(X, Y, n);
  return het::check_launch("het_gelu_fwd");
}

int het_gelu_bwd_bias(const void* dy, const void* pre, void* dpre, int64_t rows, int64_t n,
                      void* db, float* partial, void* stream) {
  if (!dy || !pre || !dpre || !db || !partial || rows < 0 || n <= 0)
    return fail(HET_EARG, "het_gelu_bwd_bias: bad args");
  if (rows == 0) {
    return cudaMemsetAsync(db, 0, n * 2, static_cast<cudaStream_t>(stream)) == cudaSuccess
               ? HET_OK
               : fail(HET_ECUDA, "het_gelu_bwd_bias: memset failed");
  }
  const bool vec = n % 8 == 0 && aligned16(dy) && aligned16(pre) && aligned16(dpre);
  GeluBwd op{static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(pre),
             static_cast<__nv_bfloat16*>(dpre)};
  return run_colsum(op, vec, rows, n, db, partial, stream, "het_gelu_bwd_bias");
}

}  // extern "C"

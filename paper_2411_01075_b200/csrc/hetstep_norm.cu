// Fused LayerNorm forward/backward for the transformer units (bf16 in/out,
// fp32 statistics). Not on the owned hot path proper, but the model's single
// largest non-GEMM cost: torch's LayerNorm backward runs a separate
// gamma/beta kernel at ~4x HBM time on [m*seq, d] bf16 activations.
//
// One warp owns a row (d = 32 * 8 * CHUNKS elements, 16-byte vectors). The
// backward is persistent: each warp walks rows with a grid stride and keeps
// its columns' dgamma/dbeta partial sums in registers; CTAs reduce their warps
// through shared memory and write one fp32 partial row each; a second pass
// sums the partial rows (fixed order: deterministic).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "hetstep.h"
#include "hetstep_internal.cuh"

using het::fail;

namespace {

constexpr int kWarps = 8;

__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 raw = *reinterpret_cast<const uint4*>(p);
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float((w[i] & 0xffffu) << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

__device__ __forceinline__ void store8(__nv_bfloat16* p, const float (&f)[8]) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int CHUNKS>
__global__ void __launch_bounds__(kWarps * 32) ln_fwd_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ r,
    const __nv_bfloat16* __restrict__ w, const __nv_bfloat16* __restrict__ b,
    __nv_bfloat16* __restrict__ xsum, __nv_bfloat16* __restrict__ y,
    float* __restrict__ mean_out, float* __restrict__ rstd_out, int64_t rows, float eps) {
  constexpr int D = CHUNKS * 256;
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  const __nv_bfloat16* xr = x + row * D;
  float v[CHUNKS][8];
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHUNKS; ++c) {
    load8(xr + c * 256 + lane * 8, v[c]);
    if (r) {                                   // residual add first: xsum = bf16(x + r)
      float rv[8];
      load8(r + row * D + c * 256 + lane * 8, rv);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        v[c][i] = __bfloat162float(__float2bfloat16_rn(v[c][i] + rv[i]));
      store8(xsum + row * D + c * 256 + lane * 8, v[c]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[c][i];
  }
  const float mean = warp_sum(s) * (1.f / D);
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < CHUNKS; ++c)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float t = v[c][i] - mean;
      q += t * t;
    }
  const float rstd = rsqrtf(warp_sum(q) * (1.f / D) + eps);
#pragma unroll
  for (int c = 0; c < CHUNKS; ++c) {
    float g[8], bb[8], o[8];
    load8(w + c * 256 + lane * 8, g);
    load8(b + c * 256 + lane * 8, bb);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = (v[c][i] - mean) * rstd * g[i] + bb[i];
    store8(y + row * D + c * 256 + lane * 8, o);
  }
  if (lane == 0) {
    mean_out[row] = mean;
    rstd_out[row] = rstd;
  }
}

template <int CHUNKS>
__global__ void __launch_bounds__(kWarps * 32, CHUNKS > 3 ? 1 : 2) ln_bwd_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ dres,
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
    const float* __restrict__ mean, const float* __restrict__ rstd,
    __nv_bfloat16* __restrict__ dx, float* __restrict__ partial /* [gridDim.x][2][D] */,
    int64_t rows) {
  constexpr int D = CHUNKS * 256;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float dg[CHUNKS][8], db[CHUNKS][8];
#pragma unroll
  for (int c = 0; c < CHUNKS; ++c)
#pragma unroll
    for (int i = 0; i < 8; ++i) dg[c][i] = db[c][i] = 0.f;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kWarps;
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * kWarps + warp; row < rows;
       row += nwarps) {
    const float mu = mean[row], rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int c = 0; c < CHUNKS; ++c) {       // pass 1: row sums + dgamma/dbeta partials
      float xv[8], dv[8], gv[8];
      load8(x + row * D + c * 256 + lane * 8, xv);
      load8(dy + row * D + c * 256 + lane * 8, dv);
      load8(w + c * 256 + lane * 8, gv);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float xh = (xv[i] - mu) * rs, gy = dv[i] * gv[i];
        dg[c][i] += dv[i] * xh;
        db[c][i] += dv[i];
        s1 += gy;
        s2 += gy * xh;
      }
    }
    s1 = warp_sum(s1) * (1.f / D);
    s2 = warp_sum(s2) * (1.f / D);
#pragma unroll
    for (int c = 0; c < CHUNKS; ++c) {       // pass 2 (row re-read from L1): dx
      float xv[8], dv[8], gv[8], o[8];
      load8(x + row * D + c * 256 + lane * 8, xv);
      load8(dy + row * D + c * 256 + lane * 8, dv);
      load8(w + c * 256 + lane * 8, gv);
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = rs * (dv[i] * gv[i] - s1 - (xv[i] - mu) * rs * s2);
      if (dres) {                              // + the residual path's gradient
        float rv[8];
        load8(dres + row * D + c * 256 + lane * 8, rv);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] += rv[i];
      }
      store8(dx + row * D + c * 256 + lane * 8, o);
    }
  }
  // CTA reduction of the warps' dgamma/dbeta partials (fixed order)
  __shared__ float red[kWarps][2][256];
#pragma unroll
  for (int c = 0; c < CHUNKS; ++c) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      red[warp][0][lane * 8 + i] = dg[c][i];
      red[warp][1][lane * 8 + i] = db[c][i];
    }
    __syncthreads();
    for (int k = threadIdx.x; k < 2 * 256; k += blockDim.x) {
      const int which = k / 256, col = k % 256;
      float acc = 0.f;
#pragma unroll
      for (int wv = 0; wv < kWarps; ++wv) acc += red[wv][which][col];
      partial[(static_cast<int64_t>(blockIdx.x) * 2 + which) * D + c * 256 + col] = acc;
    }
    __syncthreads();
  }
}

// sum the per-CTA partial rows (fixed order) -> dgamma, dbeta (bf16): a CTA owns
// 32 columns (lane = column, coalesced), its 8 warps split the partial rows and
// combine through shared memory in a fixed order.
__global__ void __launch_bounds__(256) ln_bwd_finalize_kernel(const float* __restrict__ partial,
                                                              int nblk, int64_t d,
                                                              __nv_bfloat16* __restrict__ dgamma,
                                                              __nv_bfloat16* __restrict__ dbeta) {
  __shared__ float red[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t col = static_cast<int64_t>(blockIdx.x) * 32 + lane;   // in [0, 2d)
  float acc = 0.f;
  if (col < 2 * d) {
    const int which = static_cast<int>(col / d);
    const int64_t c = col % d;
    // 8 independent partial sums per thread keep 8 loads in flight (order fixed)
    float part8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int b = warp;
    for (; b + 56 < nblk; b += 64) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        part8[k] += partial[(static_cast<int64_t>(b + 8 * k) * 2 + which) * d + c];
    }
    for (; b < nblk; b += 8) part8[0] += partial[(static_cast<int64_t>(b) * 2 + which) * d + c];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += part8[k];
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && col < 2 * d) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][lane];
    const int64_t c = col % d;
    (col / d == 0 ? dgamma : dbeta)[c] = __float2bfloat16_rn(t);
  }
}

int grid_bwd() {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms * 2;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

extern "C" {

int64_t het_layernorm_partial_floats(int64_t d) { return static_cast<int64_t>(grid_bwd()) * 2 * d; }

int het_layernorm_add_fwd(const void* x, const void* r, const void* w, const void* b, void* xsum,
                          void* y, float* mean, float* rstd, int64_t rows, int64_t d, float eps,
                          void* stream) {
  if (!x || !w || !b || !y || !mean || !rstd || rows < 0 || (d != 256 && d != 768 && d != 1024) ||
      !aligned16(x) || !aligned16(y) || !aligned16(w) || !aligned16(b) || (r && !xsum) ||
      (r && (!aligned16(r) || !aligned16(xsum))))
    return fail(HET_EARG, "het_layernorm_fwd: unsupported shape/alignment (d=%lld)", (long long)d);
  if (rows == 0) return HET_OK;
  const unsigned grid = static_cast<unsigned>((rows + kWarps - 1) / kWarps);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto X = static_cast<const __nv_bfloat16*>(x);
  auto R = static_cast<const __nv_bfloat16*>(r);
  auto W = static_cast<const __nv_bfloat16*>(w);
  auto B = static_cast<const __nv_bfloat16*>(b);
  auto S = static_cast<__nv_bfloat16*>(xsum);
  auto Y = static_cast<__nv_bfloat16*>(y);
  if (d == 256) ln_fwd_kernel<1><<<grid, kWarps * 32, 0, st>>>(X, R, W, B, S, Y, mean, rstd, rows, eps);
  else if (d == 768) ln_fwd_kernel<3><<<grid, kWarps * 32, 0, st>>>(X, R, W, B, S, Y, mean, rstd, rows, eps);
  else ln_fwd_kernel<4><<<grid, kWarps * 32, 0, st>>>(X, R, W, B, S, Y, mean, rstd, rows, eps);
  return het::check_launch("het_layernorm_fwd");
}

int het_layernorm_fwd(const void* x, const void* w, const void* b, void* y, float* mean,
                      float* rstd, int64_t rows, int64_t d, float eps, void* stream) {
  return het_layernorm_add_fwd(x, nullptr, w, b, nullptr, y, mean, rstd, rows, d, eps, stream);
}

int het_layernorm_bwd_add(const void* dy, const void* dres, const void* x, const void* w,
                          const float* mean, const float* rstd, void* dx, void* dgamma, void* dbeta,
                          float* partial, int64_t rows, int64_t d, void* stream) {
  if (!dy || !x || !w || !mean || !rstd || !dx || !dgamma || !dbeta || !partial || rows < 0 ||
      (d != 256 && d != 768 && d != 1024) || !aligned16(dy) || !aligned16(x) || !aligned16(dx) ||
      !aligned16(w) || (dres && !aligned16(dres)))
    return fail(HET_EARG, "het_layernorm_bwd: unsupported shape/alignment (d=%lld)", (long long)d);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nblk = grid_bwd();
  auto DY = static_cast<const __nv_bfloat16*>(dy);
  auto DR = static_cast<const __nv_bfloat16*>(dres);
  auto X = static_cast<const __nv_bfloat16*>(x);
  auto W = static_cast<const __nv_bfloat16*>(w);
  auto DX = static_cast<__nv_bfloat16*>(dx);
  if (d == 256) ln_bwd_kernel<1><<<nblk, kWarps * 32, 0, st>>>(DY, DR, X, W, mean, rstd, DX, partial, rows);
  else if (d == 768) ln_bwd_kernel<3><<<nblk, kWarps * 32, 0, st>>>(DY, DR, X, W, mean, rstd, DX, partial, rows);
  else ln_bwd_kernel<4><<<nblk, kWarps * 32, 0, st>>>(DY, DR, X, W, mean, rstd, DX, partial, rows);
  int rc = het::check_launch("het_layernorm_bwd");
  if (rc != HET_OK) return rc;
  ln_bwd_finalize_kernel<<<static_cast<unsigned>((2 * d + 31) / 32), 256, 0, st>>>(
      partial, nblk, d, static_cast<__nv_bfloat16*>(dgamma), static_cast<__nv_bfloat16*>(dbeta));
  return het::check_launch("het_layernorm_bwd(finalize)");
}

int het_layernorm_bwd(const void* dy, const void* x, const void* w, const float* mean,
                      const float* rstd, void* dx, void* dgamma, void* dbeta, float* partial,
                      int64_t rows, int64_t d, void* stream) {
  return het_layernorm_bwd_add(dy, nullptr, x, w, mean, rstd, dx, dgamma, dbeta, partial, rows, d,
                               stream);
}

}  // extern "C"

// ---------------------------------------------------------------- cross-entropy
//
// Fused next-token cross-entropy over bf16 logits [T, V]: the forward writes
// each row's log-sum-exp and loss (one read of the logits); the backward
// writes dlogits = scale * (softmax - onehot) in one read + one write (may
// alias the logits buffer). Replaces log_softmax + nll_loss and their
// backward (three passes over the [T, V] matrix plus the log-prob tensor).
namespace {

constexpr int kXentThreads = 512;

__device__ __forceinline__ float block_reduce(float v, bool is_max, float* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float t = __shfl_xor_sync(0xffffffffu, v, o);
    v = is_max ? fmaxf(v, t) : v + t;
  }
  if (lane == 0) smem[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < kXentThreads / 32 ? smem[lane] : (is_max ? -INFINITY : 0.f);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float t = __shfl_xor_sync(0xffffffffu, v, o);
      v = is_max ? fmaxf(v, t) : v + t;
    }
    if (lane == 0) smem[32] = v;
  }
  __syncthreads();
  const float r = smem[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kXentThreads) xent_fwd_kernel(
    const __nv_bfloat16* __restrict__ logits, const int64_t* __restrict__ target, int64_t V,
    float* __restrict__ lse_out, float* __restrict__ loss_out) {
  __shared__ float smem[33];
  const int64_t row = blockIdx.x;
  const __nv_bfloat16* x = logits + row * V;
  const int64_t nv = V / 8;
  float mx = -INFINITY, sum = 0.f;             // online max / sum of exp per thread
  for (int64_t i = threadIdx.x; i < nv; i += kXentThreads) {
    float f[8];
    load8(x + i * 8, f);
    float m8 = f[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) m8 = fmaxf(m8, f[k]);
    if (m8 > mx) {
      sum *= __expf(mx - m8);
      mx = m8;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) sum += __expf(f[k] - mx);
  }
  for (int64_t j = nv * 8 + threadIdx.x; j < V; j += kXentThreads) {
    const float v = __bfloat162float(x[j]);
    if (v > mx) {
      sum *= __expf(mx - v);
      mx = v;
    }
    sum += __expf(v - mx);
  }
  const float gmax = block_reduce(mx, true, smem);
  const float gsum = block_reduce(sum * __expf(mx - gmax), false, smem);
  if (threadIdx.x == 0) {
    const float lse = gmax + __logf(gsum);
    lse_out[row] = lse;
    loss_out[row] = lse - __bfloat162float(x[target[row]]);
  }
}

__global__ void __launch_bounds__(kXentThreads) xent_bwd_kernel(
    const __nv_bfloat16* __restrict__ logits, const int64_t* __restrict__ target, int64_t V,
    const float* __restrict__ lse, const float* __restrict__ gout, float inv_rows,
    __nv_bfloat16* __restrict__ dlogits) {
  const int64_t row = blockIdx.x;
  const float scale = *gout * inv_rows;     // upstream gradient of the mean loss
  const __nv_bfloat16* x = logits + row * V;
  __nv_bfloat16* g = dlogits + row * V;
  const float l = lse[row];
  const int64_t tgt = target[row];
  const int64_t nv = V / 8;
  for (int64_t i = threadIdx.x; i < nv; i += kXentThreads) {
    float f[8];
    load8(x + i * 8, f);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float p = __expf(f[k] - l);
      f[k] = scale * (p - (i * 8 + k == tgt ? 1.f : 0.f));
    }
    store8(g + i * 8, f);
  }
  for (int64_t j = nv * 8 + threadIdx.x; j < V; j += kXentThreads) {
    const float p = __expf(__bfloat162float(x[j]) - l);
    g[j] = __float2bfloat16_rn(scale * (p - (j == tgt ? 1.f : 0.f)));
  }
}


}  // namespace

extern "C" {


int het_xent_fwd(const void* logits, const int64_t* target, int64_t rows, int64_t vocab,
                 float* lse, float* loss, void* stream) {
  if (!logits || !target || !lse || !loss || rows < 0 || vocab <= 0 ||
      (reinterpret_cast<uintptr_t>(logits) & 15) || (vocab % 8))
    return fail(HET_EARG, "het_xent_fwd: bad args (vocab %% 8 and 16-byte alignment required)");
  if (rows == 0) return HET_OK;
  xent_fwd_kernel<<<static_cast<unsigned>(rows), kXentThreads, 0,
                    static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(logits), target, vocab, lse, loss);
  return het::check_launch("het_xent_fwd");
}

int het_xent_bwd(const void* logits, const int64_t* target, int64_t rows, int64_t vocab,
                 const float* lse, const float* grad_loss, void* dlogits, void* stream) {
  if (!logits || !target || !lse || !grad_loss || !dlogits || rows < 0 || vocab <= 0 ||
      (reinterpret_cast<uintptr_t>(logits) & 15) || (reinterpret_cast<uintptr_t>(dlogits) & 15) ||
      (vocab % 8))
    return fail(HET_EARG, "het_xent_bwd: bad args");
  if (rows == 0) return HET_OK;
  xent_bwd_kernel<<<static_cast<unsigned>(rows), kXentThreads, 0,
                    static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(logits), target, vocab, lse, grad_loss,
      1.f / static_cast<float>(rows), static_cast<__nv_bfloat16*>(dlogits));
  return het::check_launch("het_xent_bwd");
}

}  // extern "C"

// ---------------------------------------------------------------- RMSNorm + RoPE
// Llama units: y = x * rsqrt(mean(x^2) + eps) * w (fp32 math, bf16 io), and
// rotary position embedding applied in place on [rows = b*s, heads, dh]
// (rotate-half convention; backward is the inverse rotation).
namespace {

template <int CHUNKS>
__global__ void __launch_bounds__(kWarps * 32) rms_fwd_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ r,
    const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ xsum,
    __nv_bfloat16* __restrict__ y, float* __restrict__ rstd_out, int64_t rows, float eps) {
  constexpr int D = CHUNKS * 256;
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  float v[CHUNKS][8];
  float q = 0.f;
#pragma unroll
  for (int c = 0; c < CHUNKS; ++c) {
    load8(x + row * D + c * 256 + lane * 8, v[c]);
    if (r) {                                   // residual add first: xsum = bf16(x + r)
      float rv[8];
      load8(r + row * D + c * 256 + lane * 8, rv);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        v[c][i] = __bfloat162float(__float2bfloat16_rn(v[c][i] + rv[i]));
      store8(xsum + row * D + c * 256 + lane * 8, v[c]);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) q += v[c][i] * v[c][i];
  }
  const float rs = rsqrtf(warp_sum(q) * (1.f / D) + eps);
#pragma unroll
  for (int c = 0; c < CHUNKS; ++c) {
    float g[8], o[8];
    load8(w + c * 256 + lane * 8, g);
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = v[c][i] * rs * g[i];
    store8(y + row * D + c * 256 + lane * 8, o);
  }
  if (lane == 0) rstd_out[row] = rs;
}

template <int CHUNKS>
__global__ void __launch_bounds__(kWarps * 32, CHUNKS > 4 ? 1 : 2) rms_bwd_kernel(
    const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ dres,
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
    const float* __restrict__ rstd, __nv_bfloat16* __restrict__ dx,
    float* __restrict__ partial /* [gridDim.x][D] */, int64_t rows) {
  constexpr int D = CHUNKS * 256;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float dg[CHUNKS][8];
#pragma unroll
  for (int c = 0; c < CHUNKS; ++c)
#pragma unroll
    for (int i = 0; i < 8; ++i) dg[c][i] = 0.f;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kWarps;
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * kWarps + warp; row < rows;
       row += nwarps) {
    const float rs = rstd[row];
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < CHUNKS; ++c) {
      float xv[8], dv[8], gv[8];
      load8(x + row * D + c * 256 + lane * 8, xv);
      load8(dy + row * D + c * 256 + lane * 8, dv);
      load8(w + c * 256 + lane * 8, gv);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float xh = xv[i] * rs;
        dg[c][i] += dv[i] * xh;
        s += dv[i] * gv[i] * xh;
      }
    }
    s = warp_sum(s) * (1.f / D);
#pragma unroll
    for (int c = 0; c < CHUNKS; ++c) {
      float xv[8], dv[8], gv[8], o[8];
      load8(x + row * D + c * 256 + lane * 8, xv);
      load8(dy + row * D + c * 256 + lane * 8, dv);
      load8(w + c * 256 + lane * 8, gv);
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = rs * (dv[i] * gv[i] - xv[i] * rs * s);
      if (dres) {                              // + the residual path's gradient
        float rv[8];
        load8(dres + row * D + c * 256 + lane * 8, rv);
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] += rv[i];
      }
      store8(dx + row * D + c * 256 + lane * 8, o);
    }
  }
  __shared__ float red[kWarps][256];
#pragma unroll
  for (int c = 0; c < CHUNKS; ++c) {
#pragma unroll
    for (int i = 0; i < 8; ++i) red[warp][lane * 8 + i] = dg[c][i];
    __syncthreads();
    for (int k = threadIdx.x; k < 256; k += blockDim.x) {
      float acc = 0.f;
#pragma unroll
      for (int wv = 0; wv < kWarps; ++wv) acc += red[wv][k];
      partial[static_cast<int64_t>(blockIdx.x) * D + c * 256 + k] = acc;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) rms_bwd_finalize_kernel(const float* __restrict__ partial,
                                                               int nblk, int64_t d,
                                                               __nv_bfloat16* __restrict__ dgamma) {
  __shared__ float red[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t col = static_cast<int64_t>(blockIdx.x) * 32 + lane;
  float part8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (col < d) {
    int b = warp;
    for (; b + 56 < nblk; b += 64) {
#pragma unroll
      for (int k = 0; k < 8; ++k) part8[k] += partial[static_cast<int64_t>(b + 8 * k) * d + col];
    }
    for (; b < nblk; b += 8) part8[0] += partial[static_cast<int64_t>(b) * d + col];
  }
  float acc = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc += part8[k];
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && col < d) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][lane];
    dgamma[col] = __float2bfloat16_rn(t);
  }
}

// x: [rows, heads, dh] bf16 contiguous, position of row r = r % seq; rotate
// pairs (i, i + dh/2) by angle pos * 10000^(-2i/dh) (sign = -1 for backward)
__global__ void rope_kernel(__nv_bfloat16* __restrict__ x, int64_t rows, int heads, int dh,
                            int64_t seq, float sign) {
  const int half = dh / 2;
  const int64_t total = rows * heads * half;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += stride) {
    const int i = static_cast<int>(t % half);
    const int64_t rh = t / half;                      // row * heads + head
    const int64_t pos = (rh / heads) % seq;
    const float inv = exp2f(-static_cast<float>(2 * i) / dh * 13.287712379549449f);  // log2(1e4)
    float sn, cs;
    __sincosf(static_cast<float>(pos) * inv, &sn, &cs);
    sn *= sign;
    __nv_bfloat16* p = x + rh * dh;
    const float a = __bfloat162float(p[i]), b = __bfloat162float(p[i + half]);
    p[i] = __float2bfloat16_rn(a * cs - b * sn);
    p[i + half] = __float2bfloat16_rn(a * sn + b * cs);
  }
}

// ---------------------------------------------------------------- SwiGLU
// out = silu(a) * b on bf16 [rows, f] (a, b with row stride ld); the rounding
// sequence of torch's two-kernel form (silu rounded to bf16, then the product)
// so the fused pass reproduces F.silu(a) * b. 8 elements per thread per step
// (16-byte accesses) when f and the strides allow it.
__device__ __forceinline__ float silu_f(float a) { return a / (1.0f + expf(-a)); }
__device__ __forceinline__ float rbf(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

template <int V>
__global__ void swiglu_fwd_kernel(const __nv_bfloat16* __restrict__ a,
                                  const __nv_bfloat16* __restrict__ b, int64_t ld,
                                  __nv_bfloat16* __restrict__ out, int64_t rows, int64_t f) {
  const int64_t per_row = f / V;
  const int64_t total = rows * per_row;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += stride) {
    const int64_t r = t / per_row, c = (t - r * per_row) * V;
    __nv_bfloat16 av[V], bv[V], ov[V];
    if (V == 8) {
      *reinterpret_cast<uint4*>(av) = __ldcs(reinterpret_cast<const uint4*>(a + r * ld + c));
      *reinterpret_cast<uint4*>(bv) = __ldcs(reinterpret_cast<const uint4*>(b + r * ld + c));
    } else {
      av[0] = a[r * ld + c];
      bv[0] = b[r * ld + c];
    }
#pragma unroll
    for (int i = 0; i < V; ++i)
      ov[i] = __float2bfloat16_rn(rbf(silu_f(__bfloat162float(av[i]))) * __bfloat162float(bv[i]));
    if (V == 8)
      *reinterpret_cast<uint4*>(out + r * f + c) = *reinterpret_cast<uint4*>(ov);
    else
      out[r * f + c] = ov[0];
  }
}

// da = (g*b) * s * (1 + a (1 - s)), db = g * silu(a), s = sigmoid(a) (torch's
// mul / silu backward, g*b rounded to bf16 in between as torch does)
template <int V>
__global__ void swiglu_bwd_kernel(const __nv_bfloat16* __restrict__ g,
                                  const __nv_bfloat16* __restrict__ a,
                                  const __nv_bfloat16* __restrict__ b, int64_t ld,
                                  __nv_bfloat16* __restrict__ da, __nv_bfloat16* __restrict__ db,
                                  int64_t ldg, int64_t rows, int64_t f) {
  const int64_t per_row = f / V;
  const int64_t total = rows * per_row;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += stride) {
    const int64_t r = t / per_row, c = (t - r * per_row) * V;
    __nv_bfloat16 gv[V], av[V], bv[V], dav[V], dbv[V];
    if (V == 8) {
      *reinterpret_cast<uint4*>(gv) = __ldcs(reinterpret_cast<const uint4*>(g + r * f + c));
      *reinterpret_cast<uint4*>(av) = __ldcs(reinterpret_cast<const uint4*>(a + r * ld + c));
      *reinterpret_cast<uint4*>(bv) = __ldcs(reinterpret_cast<const uint4*>(b + r * ld + c));
    } else {
      gv[0] = g[r * f + c];
      av[0] = a[r * ld + c];
      bv[0] = b[r * ld + c];
    }
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const float x = __bfloat162float(av[i]), gg = __bfloat162float(gv[i]);
      const float s = 1.0f / (1.0f + expf(-x));
      const float dsilu = rbf(gg * __bfloat162float(bv[i]));
      dav[i] = __float2bfloat16_rn(dsilu * s * (1.0f + x * (1.0f - s)));
      dbv[i] = __float2bfloat16_rn(gg * rbf(silu_f(x)));
    }
    if (V == 8) {
      *reinterpret_cast<uint4*>(da + r * ldg + c) = *reinterpret_cast<uint4*>(dav);
      *reinterpret_cast<uint4*>(db + r * ldg + c) = *reinterpret_cast<uint4*>(dbv);
    } else {
      da[r * ldg + c] = dav[0];
      db[r * ldg + c] = dbv[0];
    }
  }
}

unsigned elementwise_grid(int64_t items, int threads) {
  int64_t blocks = (items + threads - 1) / threads;
  const int64_t cap = 148 * 8;                  // grid-stride: 8 CTAs of 256 per SM
  return static_cast<unsigned>(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}


// Fused q/k/v projection output [rows, 3 * heads * dh] -> rotary-embedded q, k and a
// copy of v, each contiguous [rows, heads, dh] (MERGE = false), or the backward:
// dq, dk (inverse rotation) and dv back into one [rows, 3 * heads * dh] gradient
// (MERGE = true). One thread per (row, head, 8-pair group): 16-byte accesses.
template <bool MERGE>
__global__ void rope_qkv_kernel(const __nv_bfloat16* __restrict__ in0,
                                const __nv_bfloat16* __restrict__ in1,
                                const __nv_bfloat16* __restrict__ in2,
                                __nv_bfloat16* __restrict__ out0, __nv_bfloat16* __restrict__ out1,
                                __nv_bfloat16* __restrict__ out2, int64_t rows, int heads, int dh,
                                int64_t seq) {
  const int half = dh / 2, groups = half / 8;
  const int64_t d = static_cast<int64_t>(heads) * dh;
  const int64_t total = rows * heads * groups;
  const float sign = MERGE ? -1.f : 1.f;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
       t += stride) {
    const int gi = static_cast<int>(t % groups);
    const int64_t rh = t / groups;                 // row * heads + head
    const int64_t row = rh / heads;
    const int head = static_cast<int>(rh - row * heads);
    const int64_t pos = row % seq;
    const int64_t packed = row * 3 * d + static_cast<int64_t>(head) * dh;   // q slot in [rows, 3d]
    const int64_t split = row * d + static_cast<int64_t>(head) * dh;        // in [rows, d]
    const int i0 = gi * 8;
#pragma unroll
    for (int which = 0; which < 2; ++which) {      // q, k
      const __nv_bfloat16* src = MERGE ? (which ? in1 : in0) + split : in0 + packed + which * d;
      __nv_bfloat16* dst = MERGE ? out0 + packed + which * d : (which ? out1 : out0) + split;
      __nv_bfloat16 lo[8], hi[8], ol[8], oh[8];
      *reinterpret_cast<uint4*>(lo) = *reinterpret_cast<const uint4*>(src + i0);
      *reinterpret_cast<uint4*>(hi) = *reinterpret_cast<const uint4*>(src + i0 + half);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = i0 + j;
        const float inv = exp2f(-static_cast<float>(2 * i) / dh * 13.287712379549449f);
        float sn, cs;
        __sincosf(static_cast<float>(pos) * inv, &sn, &cs);
        sn *= sign;
        const float a = __bfloat162float(lo[j]), b = __bfloat162float(hi[j]);
        ol[j] = __float2bfloat16_rn(a * cs - b * sn);
        oh[j] = __float2bfloat16_rn(a * sn + b * cs);
      }
      *reinterpret_cast<uint4*>(dst + i0) = *reinterpret_cast<const uint4*>(ol);
      *reinterpret_cast<uint4*>(dst + i0 + half) = *reinterpret_cast<const uint4*>(oh);
    }
    // v: plain copy of this thread's 2 x 8 elements
    const __nv_bfloat16* vs = MERGE ? in2 + split : in0 + packed + 2 * d;
    __nv_bfloat16* vd = MERGE ? out0 + packed + 2 * d : out2 + split;
    *reinterpret_cast<uint4*>(vd + i0) = *reinterpret_cast<const uint4*>(vs + i0);
    *reinterpret_cast<uint4*>(vd + i0 + half) = *reinterpret_cast<const uint4*>(vs + i0 + half);
  }
}
}  // namespace

extern "C" {

int64_t het_rmsnorm_partial_floats(int64_t d) { return static_cast<int64_t>(grid_bwd()) * d; }

int het_rmsnorm_add_fwd(const void* x, const void* r, const void* w, void* xsum, void* y,
                        float* rstd, int64_t rows, int64_t d, float eps, void* stream) {
  if (!x || !w || !y || !rstd || rows < 0 || (d != 2048 && d != 1024 && d != 768 && d != 256) ||
      !aligned16(x) || !aligned16(y) || !aligned16(w) || (r && !xsum) ||
      (r && (!aligned16(r) || !aligned16(xsum))))
    return fail(HET_EARG, "het_rmsnorm_fwd: unsupported shape/alignment (d=%lld)", (long long)d);
  if (rows == 0) return HET_OK;
  const unsigned grid = static_cast<unsigned>((rows + kWarps - 1) / kWarps);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto X = static_cast<const __nv_bfloat16*>(x);
  auto R = static_cast<const __nv_bfloat16*>(r);
  auto W = static_cast<const __nv_bfloat16*>(w);
  auto S = static_cast<__nv_bfloat16*>(xsum);
  auto Y = static_cast<__nv_bfloat16*>(y);
  switch (d) {
    case 256: rms_fwd_kernel<1><<<grid, kWarps * 32, 0, st>>>(X, R, W, S, Y, rstd, rows, eps); break;
    case 768: rms_fwd_kernel<3><<<grid, kWarps * 32, 0, st>>>(X, R, W, S, Y, rstd, rows, eps); break;
    case 1024: rms_fwd_kernel<4><<<grid, kWarps * 32, 0, st>>>(X, R, W, S, Y, rstd, rows, eps); break;
    default: rms_fwd_kernel<8><<<grid, kWarps * 32, 0, st>>>(X, R, W, S, Y, rstd, rows, eps);
  }
  return het::check_launch("het_rmsnorm_fwd");
}

int het_rmsnorm_fwd(const void* x, const void* w, void* y, float* rstd, int64_t rows, int64_t d,
                    float eps, void* stream) {
  return het_rmsnorm_add_fwd(x, nullptr, w, nullptr, y, rstd, rows, d, eps, stream);
}

int het_rmsnorm_bwd_add(const void* dy, const void* dres, const void* x, const void* w,
                        const float* rstd, void* dx, void* dgamma, float* partial, int64_t rows,
                        int64_t d, void* stream) {
  if (!dy || !x || !w || !rstd || !dx || !dgamma || !partial || rows < 0 ||
      (d != 2048 && d != 1024 && d != 768 && d != 256) || !aligned16(dy) || !aligned16(x) ||
      !aligned16(dx) || !aligned16(w) || (dres && !aligned16(dres)))
    return fail(HET_EARG, "het_rmsnorm_bwd: unsupported shape/alignment (d=%lld)", (long long)d);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nblk = grid_bwd();
  auto DY = static_cast<const __nv_bfloat16*>(dy);
  auto DR = static_cast<const __nv_bfloat16*>(dres);
  auto X = static_cast<const __nv_bfloat16*>(x);
  auto W = static_cast<const __nv_bfloat16*>(w);
  auto DX = static_cast<__nv_bfloat16*>(dx);
  switch (d) {
    case 256: rms_bwd_kernel<1><<<nblk, kWarps * 32, 0, st>>>(DY, DR, X, W, rstd, DX, partial, rows); break;
    case 768: rms_bwd_kernel<3><<<nblk, kWarps * 32, 0, st>>>(DY, DR, X, W, rstd, DX, partial, rows); break;
    case 1024: rms_bwd_kernel<4><<<nblk, kWarps * 32, 0, st>>>(DY, DR, X, W, rstd, DX, partial, rows); break;
    default: rms_bwd_kernel<8><<<nblk, kWarps * 32, 0, st>>>(DY, DR, X, W, rstd, DX, partial, rows);
  }
  int rc = het::check_launch("het_rmsnorm_bwd");
  if (rc != HET_OK) return rc;
  rms_bwd_finalize_kernel<<<static_cast<unsigned>((d + 31) / 32), 256, 0, st>>>(
      partial, nblk, d, static_cast<__nv_bfloat16*>(dgamma));
  return het::check_launch("het_rmsnorm_bwd(finalize)");
}

int het_rmsnorm_bwd(const void* dy, const void* x, const void* w, const float* rstd, void* dx,
                    void* dgamma, float* partial, int64_t rows, int64_t d, void* stream) {
  return het_rmsnorm_bwd_add(dy, nullptr, x, w, rstd, dx, dgamma, partial, rows, d, stream);
}

int het_rope_inplace(void* x, int64_t rows, int heads, int dh, int64_t seq, int inverse,
                     void* stream) {
  if (!x || rows < 0 || heads <= 0 || dh <= 0 || (dh % 2) || seq <= 0)
    return fail(HET_EARG, "het_rope_inplace: bad args");
  const int64_t total = rows * heads * (dh / 2);
  if (total == 0) return HET_OK;
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  rope_kernel<<<static_cast<unsigned>(blocks), threads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<__nv_bfloat16*>(x), rows, heads, dh, seq, inverse ? -1.f : 1.f);
  return het::check_launch("het_rope_inplace");
}

int het_swiglu_fwd(const void* a, const void* b, int64_t ld, void* out, int64_t rows, int64_t f,
                   void* stream) {
  if (!a || !b || !out || rows < 0 || f <= 0 || ld < f)
    return fail(HET_EARG, "het_swiglu_fwd: bad args");
  if (rows == 0) return HET_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto A = static_cast<const __nv_bfloat16*>(a);
  auto B = static_cast<const __nv_bfloat16*>(b);
  auto O = static_cast<__nv_bfloat16*>(out);
  if (f % 8 == 0 && ld % 8 == 0 && aligned16(a) && aligned16(b) && aligned16(out))
    swiglu_fwd_kernel<8><<<elementwise_grid(rows * f / 8, 256), 256, 0, st>>>(A, B, ld, O, rows, f);
  else
    swiglu_fwd_kernel<1><<<elementwise_grid(rows * f, 256), 256, 0, st>>>(A, B, ld, O, rows, f);
  return het::check_launch("het_swiglu_fwd");
}

int het_swiglu_bwd(const void* dout, const void* a, const void* b, int64_t ld, void* da, void* db,
                   int64_t ldg, int64_t rows, int64_t f, void* stream) {
  if (!dout || !a || !b || !da || !db || rows < 0 || f <= 0 || ld < f || ldg < f)
    return fail(HET_EARG, "het_swiglu_bwd: bad args");
  if (rows == 0) return HET_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto G = static_cast<const __nv_bfloat16*>(dout);
  auto A = static_cast<const __nv_bfloat16*>(a);
  auto B = static_cast<const __nv_bfloat16*>(b);
  auto DA = static_cast<__nv_bfloat16*>(da);
  auto DB = static_cast<__nv_bfloat16*>(db);
  if (f % 8 == 0 && ld % 8 == 0 && ldg % 8 == 0 && aligned16(dout) && aligned16(a) &&
      aligned16(b) && aligned16(da) && aligned16(db))
    swiglu_bwd_kernel<8><<<elementwise_grid(rows * f / 8, 256), 256, 0, st>>>(G, A, B, ld, DA, DB,
                                                                             ldg, rows, f);
  else
    swiglu_bwd_kernel<1><<<elementwise_grid(rows * f, 256), 256, 0, st>>>(G, A, B, ld, DA, DB, ldg,
                                                                         rows, f);
  return het::check_launch("het_swiglu_bwd");
}

int het_rope_qkv_split(const void* qkv, void* q, void* k, void* v, int64_t rows, int heads, int dh,
                       int64_t seq, void* stream) {
  if (!qkv || !q || !k || !v || rows < 0 || heads <= 0 || dh <= 0 || dh % 16 || seq <= 0 ||
      !aligned16(qkv) || !aligned16(q) || !aligned16(k) || !aligned16(v))
    return fail(HET_EARG, "het_rope_qkv_split: bad args (dh %% 16, 16-byte alignment)");
  const int64_t total = rows * heads * (dh / 16);
  if (total == 0) return HET_OK;
  rope_qkv_kernel<false><<<elementwise_grid(total, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(qkv), nullptr, nullptr, static_cast<__nv_bfloat16*>(q),
      static_cast<__nv_bfloat16*>(k), static_cast<__nv_bfloat16*>(v), rows, heads, dh, seq);
  return het::check_launch("het_rope_qkv_split");
}

int het_rope_qkv_merge(const void* dq, const void* dk, const void* dv, void* dqkv, int64_t rows,
                       int heads, int dh, int64_t seq, void* stream) {
  if (!dq || !dk || !dv || !dqkv || rows < 0 || heads <= 0 || dh <= 0 || dh % 16 || seq <= 0 ||
      !aligned16(dq) || !aligned16(dk) || !aligned16(dv) || !aligned16(dqkv))
    return fail(HET_EARG, "het_rope_qkv_merge: bad args (dh %% 16, 16-byte alignment)");
  const int64_t total = rows * heads * (dh / 16);
  if (total == 0) return HET_OK;
  rope_qkv_kernel<true><<<elementwise_grid(total, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(dq), static_cast<const __nv_bfloat16*>(dk),
      static_cast<const __nv_bfloat16*>(dv), static_cast<__nv_bfloat16*>(dqkv), nullptr, nullptr,
      rows, heads, dh, seq);
  return het::check_launch("het_rope_qkv_merge");
}

}  // extern "C"

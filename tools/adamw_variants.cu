// Micro-benchmark of AdamW / accumulate memory-access variants on one B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o adamw_variants tools/adamw_variants.cu
//   ./adamw_variants [n_elements]
// Prints achieved algorithmic GB/s (28 B/param AdamW without shadow, 30 with)
// for: 128-bit x2 unroll (current), 256-bit (ld/st.global.v8), 256-bit x2,
// and a 256-bit copy as the practical stream ceiling.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

struct C { float decay, omb1, b2, omb2, bc2s, eps, neg; };

__device__ __forceinline__ void adam1(float& p, float g, float& m, float& v, const C& c) {
  p = __fmul_rn(p, c.decay);
  m = __fmaf_rn(c.omb1, __fsub_rn(g, m), m);
  v = __fmaf_rn(__fmul_rn(c.omb2, g), g, __fmul_rn(v, c.b2));
  const float d = __fadd_rn(__fdiv_rn(__fsqrt_rn(v), c.bc2s), c.eps);
  p = __fmaf_rn(c.neg, __fdiv_rn(m, d), p);
}

struct F8 { float x[8]; };
__device__ __forceinline__ F8 ld8(const float* a) {
  F8 r;
  asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]),
                 "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7]) : "l"(a));
  return r;
}
__device__ __forceinline__ F8 ld8cs(const float* a) {
  F8 r;
  asm volatile("ld.global.cs.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.x[0]), "=f"(r.x[1]), "=f"(r.x[2]), "=f"(r.x[3]), "=f"(r.x[4]),
                 "=f"(r.x[5]), "=f"(r.x[6]), "=f"(r.x[7]) : "l"(a));
  return r;
}
__device__ __forceinline__ void st8(float* a, const F8& r) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" :: "l"(a),
               "f"(r.x[0]), "f"(r.x[1]), "f"(r.x[2]), "f"(r.x[3]), "f"(r.x[4]), "f"(r.x[5]),
               "f"(r.x[6]), "f"(r.x[7]) : "memory");
}

__global__ void adam_v4x2(float4* p, const float4* g, float4* m, float4* v, int64_t n4, C c) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += 2 * st) {
    const int64_t j = i + st; const bool two = j < n4;
    float4 p0 = p[i], g0 = __ldcs(g + i), m0 = m[i], v0 = v[i], p1, g1, m1, v1;
    if (two) { p1 = p[j]; g1 = __ldcs(g + j); m1 = m[j]; v1 = v[j]; }
    adam1(p0.x, g0.x, m0.x, v0.x, c); adam1(p0.y, g0.y, m0.y, v0.y, c);
    adam1(p0.z, g0.z, m0.z, v0.z, c); adam1(p0.w, g0.w, m0.w, v0.w, c);
    p[i] = p0; m[i] = m0; v[i] = v0;
    if (two) {
      adam1(p1.x, g1.x, m1.x, v1.x, c); adam1(p1.y, g1.y, m1.y, v1.y, c);
      adam1(p1.z, g1.z, m1.z, v1.z, c); adam1(p1.w, g1.w, m1.w, v1.w, c);
      p[j] = p1; m[j] = m1; v[j] = v1;
    }
  }
}

template <int U, bool CS>
__global__ void adam_v8(float* p, const float* g, float* m, float* v, int64_t n8, C c) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n8; i0 += U * st) {
    F8 P[U], G[U], M[U], V[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * st;
      if (i < n8) {
        P[u] = ld8(p + i * 8); G[u] = CS ? ld8cs(g + i * 8) : ld8(g + i * 8);
        M[u] = ld8(m + i * 8); V[u] = ld8(v + i * 8);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * st;
      if (i < n8) {
#pragma unroll
        for (int k = 0; k < 8; ++k) adam1(P[u].x[k], G[u].x[k], M[u].x[k], V[u].x[k], c);
        st8(p + i * 8, P[u]); st8(m + i * 8, M[u]); st8(v + i * 8, V[u]);
      }
    }
  }
}

__global__ void copy_v8(const float* a, float* b, int64_t n8) {
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += st)
    st8(b + i * 8, ld8(a + i * 8));
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 124082688;
  float *p, *g, *m, *v;
  CK(cudaMalloc(&p, n * 4)); CK(cudaMalloc(&g, n * 4)); CK(cudaMalloc(&m, n * 4)); CK(cudaMalloc(&v, n * 4));
  CK(cudaMemset(p, 0, n * 4)); CK(cudaMemset(g, 0, n * 4)); CK(cudaMemset(m, 0, n * 4)); CK(cudaMemset(v, 0, n * 4));
  C c{0.9999f, 0.1f, 0.95f, 0.05f, 0.3f, 1e-8f, -1e-3f};
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](const char* name, double bytes, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
    }
    printf("%-28s %8.3f ms  %8.1f GB/s\n", name, best, bytes / (best * 1e-3) / 1e9);
  };
  const double ab = 28.0 * n;
  for (int threads : {256, 512}) {
    for (int mult : {4, 8, 16}) {
      int grid = sms * mult * 256 / threads;
      char nm[64];
      snprintf(nm, sizeof nm, "v4x2 t%d g%dx", threads, mult);
      run(nm, ab, [&] { adam_v4x2<<<grid, threads>>>((float4*)p, (float4*)g, (float4*)m, (float4*)v, n / 4, c); });
      snprintf(nm, sizeof nm, "v8x1 t%d g%dx", threads, mult);
      run(nm, ab, [&] { adam_v8<1, true><<<grid, threads>>>(p, g, m, v, n / 8, c); });
      snprintf(nm, sizeof nm, "v8x2 t%d g%dx", threads, mult);
      run(nm, ab, [&] { adam_v8<2, true><<<grid, threads>>>(p, g, m, v, n / 8, c); });
    }
  }
  run("copy v8 (2 streams)", 8.0 * n, [&] { copy_v8<<<sms * 8, 256>>>(p, m, n / 8); });
  run("cudaMemcpy D2D", 8.0 * n, [&] { cudaMemcpyAsync(m, p, n * 4, cudaMemcpyDeviceToDevice); });
  return 0;
}

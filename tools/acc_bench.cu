// Per-launch device time of het_accumulate shape variants through the C-ABI.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Iinclude tools/acc_bench.cu \
//        -Lpaper_2411_01075_b200/_lib -lhetstep -Xlinker -rpath=$PWD/paper_2411_01075_b200/_lib \
//        -o tools/acc_bench && ./tools/acc_bench
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>
#include "hetstep.h"

int main() {
  const long sizes[] = {789760, 7087872, 12596224, 51384320};
  void* flush;
  cudaMalloc(&flush, 512 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (long n : sizes) {
    void* g;
    float* acc;
    cudaMalloc(&g, n * 2);
    cudaMalloc(&acc, n * 4);
    cudaMemset(g, 0, n * 2);
    het_seg_t seg{g, 0, n};
    for (int v = 0; v < 6; ++v) {
      het_tune(HET_TUNE_ACC_VARIANT, v);
      for (int mode = 1; mode >= 0; --mode) {
        for (int cold = 0; cold < 2; ++cold) {
          std::vector<float> t;
          for (int r = 0; r < 12; ++r) {
            if (cold) cudaMemsetAsync(flush, r, 512 << 20);
            cudaEventRecord(a);
            het_accumulate(acc, &seg, 1, mode, 0.5f, nullptr);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            t.push_back(ms);
          }
          std::sort(t.begin() + 2, t.end());
          const float med = t[2 + (t.size() - 2) / 2];
          const double bytes = (mode ? 6.0 : 10.0) * n;
          printf("n=%9ld variant=%d %s %s  %8.2f us  %7.1f GB/s\n", n, v, mode ? "FIRST" : "ADD  ",
                 cold ? "cold" : "hot ", med * 1e3, bytes / (med * 1e-3) / 1e9);
        }
      }
    }
    cudaFree(g);
    cudaFree(acc);
  }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

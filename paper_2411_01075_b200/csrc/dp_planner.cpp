// Native core of the batch-assignment dynamic program.
//
// One call processes one GPU layer of the DP: given the previous slab
// prev[j][k] (best max-latency with j samples and microbatch mass k assigned
// to the GPUs before this one) and this GPU's transition list (m, T(m,l) for
// l = 1..), it fills cur[j][k] and the (m, l) choice planes.
//
// Semantics are those of the reference DP (pkg/src/hetplan/planner.py:448-477):
// every cell takes the FIRST strict improvement while transitions are scanned
// in ascending (m, l) order, so ties resolve to the lexicographically smallest
// (m, l). Because each transition reads only `prev`, scanning transitions in
// order per row block is equivalent to the reference's slab-at-a-time update,
// and the result is bit-identical for any thread count.
//
// Host-only C++ (g++), no CUDA: the planner runs once per job, offline.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <thread>
#include <vector>

namespace {

struct RowSpan {
  int lo, hi;  // finite k range [lo, hi], lo > hi when the row is empty
};

void update_rows(const double* prev, double* cur, int16_t* cm, int16_t* cl,
                 const int32_t* opt_m, const int32_t* opt_len, const int64_t* opt_off,
                 const double* opt_t, int n_opts, int size, const RowSpan* span,
                 int r0, int r1) {
  for (int o = 0; o < n_opts; ++o) {
    const int m = opt_m[o];
    const double* t_arr = opt_t + opt_off[o];
    for (int li = 0; li < opt_len[o]; ++li) {
      const int b = m * (li + 1);
      const int lo = std::max(r0, b);
      if (lo >= r1) break;
      const double t = t_arr[li];
      const int16_t mm = static_cast<int16_t>(m), ll = static_cast<int16_t>(li + 1);
      for (int j = lo; j < r1; ++j) {
        const RowSpan s = span[j - b];
        if (s.lo > s.hi) continue;
        // source columns k-m in [s.lo, s.hi]  ->  target k in [s.lo+m, s.hi+m] ∩ [m, size)
        const int k0 = s.lo + m;
        const int k1 = std::min(s.hi + m, size - 1);
        const double* src = prev + static_cast<int64_t>(j - b) * size;
        double* dst = cur + static_cast<int64_t>(j) * size;
        int16_t* dm = cm + static_cast<int64_t>(j) * size;
        int16_t* dl = cl + static_cast<int64_t>(j) * size;
        for (int k = k0; k <= k1; ++k) {
          const double p = src[k - m];
          const double cand = p > t ? p : t;  // np.maximum (no NaNs reach here)
          if (cand < dst[k]) {
            dst[k] = cand;
            dm[k] = mm;
            dl[k] = ll;
          }
        }
      }
    }
  }
}

}  // namespace

extern "C" {

// Returns 0 on success. prev/cur are size*size row-major doubles; cur, cm, cl
// must already hold their initial values (inf/-1, or prev/0 with idle allowed).
int het_dp_layer(const double* prev, double* cur, int16_t* cm, int16_t* cl,
                 const int32_t* opt_m, const int32_t* opt_len, const int64_t* opt_off,
                 const double* opt_t, int n_opts, int size, int threads) {
  if (size <= 0 || n_opts < 0) return 1;
  std::vector<RowSpan> span(size);
  for (int r = 0; r < size; ++r) {
    const double* row = prev + static_cast<int64_t>(r) * size;
    int lo = size, hi = -1;
    for (int k = 0; k < size; ++k) {
      if (std::isfinite(row[k])) {
        lo = std::min(lo, k);
        hi = k;
      }
    }
    span[r] = {lo, hi};
  }
  if (threads <= 1 || size < 64) {
    update_rows(prev, cur, cm, cl, opt_m, opt_len, opt_off, opt_t, n_opts, size,
                span.data(), 0, size);
    return 0;
  }
  // interleaved row blocks balance the triangular (k <= j) work
  const int block = 8;
  const int nblocks = (size + block - 1) / block;
  std::vector<std::thread> pool;
  for (int w = 0; w < threads; ++w) {
    pool.emplace_back([&, w]() {
      for (int bi = w; bi < nblocks; bi += threads) {
        const int r0 = bi * block, r1 = std::min(size, r0 + block);
        update_rows(prev, cur, cm, cl, opt_m, opt_len, opt_off, opt_t, n_opts, size,
                    span.data(), r0, r1);
      }
    });
  }
  for (auto& th : pool) th.join();
  return 0;
}

}  // extern "C"

// Library GEMMs with fused epilogues through cuBLASLt, for the model's linear
// layers (bf16 operands, fp32 compute): bias, GELU (+ the pre-activation kept
// for the backward), and in the backward the GELU derivative and the bias
// gradients, so the step needs no separate GELU / bias-reduction passes.
// cuBLASLt's own kernels run the math; this file only owns the descriptors,
// a per-shape plan cache and the C-ABI.
#include <cublasLt.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <tuple>
#include <unordered_map>

#include "hetstep.h"
#include "hetstep_internal.cuh"

using het::fail;

namespace {

struct Key {
  int ta, tb, epi;
  int64_t m, n, k, lda, ldb, ldd, ldaux;
  int device;
  bool operator==(const Key& o) const {
    return std::tie(ta, tb, epi, m, n, k, lda, ldb, ldd, ldaux, device) ==
           std::tie(o.ta, o.tb, o.epi, o.m, o.n, o.k, o.lda, o.ldb, o.ldd, o.ldaux, o.device);
  }
};

struct KeyHash {
  size_t operator()(const Key& k) const {
    size_t h = 1469598103934665603ull;
    const int64_t v[] = {k.ta, k.tb, k.epi, k.m, k.n, k.k, k.lda, k.ldb, k.ldd, k.ldaux, k.device};
    for (int64_t x : v) h = (h ^ static_cast<size_t>(x)) * 1099511628211ull;
    return h;
  }
};

struct Plan {
  cublasLtMatmulDesc_t desc = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, d = nullptr;
  cublasLtMatmulAlgo_t algo;
  size_t ws = 0;
};

std::mutex g_mu;
std::unordered_map<Key, Plan, KeyHash> g_plans;
cublasLtHandle_t g_handle[16] = {};

cublasLtEpilogue_t epilogue_of(int e) {
  switch (e) {
    case HET_LT_BIAS: return CUBLASLT_EPILOGUE_BIAS;
    case HET_LT_GELU_BIAS: return CUBLASLT_EPILOGUE_GELU_BIAS;
    case HET_LT_GELU_AUX_BIAS: return CUBLASLT_EPILOGUE_GELU_AUX_BIAS;
    case HET_LT_DGELU_BGRAD: return CUBLASLT_EPILOGUE_DGELU_BGRAD;
    case HET_LT_BGRADB: return CUBLASLT_EPILOGUE_BGRADB;
    default: return CUBLASLT_EPILOGUE_DEFAULT;
  }
}

#define LT_CHECK(x, what)                                                        \
  do {                                                                           \
    cublasStatus_t st_ = (x);                                                    \
    if (st_ != CUBLAS_STATUS_SUCCESS)                                            \
      return fail(HET_ECUDA, "het_lt_matmul: %s failed (status %d)", what, (int)st_); \
  } while (0)

int make_plan(const Key& k, cublasLtHandle_t h, size_t ws_cap, Plan* out) {
  Plan p;
  LT_CHECK(cublasLtMatmulDescCreate(&p.desc, CUBLAS_COMPUTE_32F, CUDA_R_32F), "DescCreate");
  const cublasOperation_t ta = k.ta ? CUBLAS_OP_T : CUBLAS_OP_N;
  const cublasOperation_t tb = k.tb ? CUBLAS_OP_T : CUBLAS_OP_N;
  LT_CHECK(cublasLtMatmulDescSetAttribute(p.desc, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)),
           "TRANSA");
  LT_CHECK(cublasLtMatmulDescSetAttribute(p.desc, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)),
           "TRANSB");
  const cublasLtEpilogue_t epi = epilogue_of(k.epi);
  LT_CHECK(cublasLtMatmulDescSetAttribute(p.desc, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi)),
           "EPILOGUE");
  if (k.epi != HET_LT_NONE) {
    const cudaDataType_t bt = CUDA_R_16BF;
    LT_CHECK(cublasLtMatmulDescSetAttribute(p.desc, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bt,
                                            sizeof(bt)), "BIAS_DATA_TYPE");
  }
  if (k.epi == HET_LT_GELU_AUX_BIAS || k.epi == HET_LT_DGELU_BGRAD) {
    const int64_t ld = k.ldaux;
    LT_CHECK(cublasLtMatmulDescSetAttribute(p.desc, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_LD, &ld,
                                            sizeof(ld)), "AUX_LD");
    const cudaDataType_t at = CUDA_R_16BF;
    LT_CHECK(cublasLtMatmulDescSetAttribute(p.desc, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_DATA_TYPE,
                                            &at, sizeof(at)), "AUX_DATA_TYPE");
  }
  // column-major layouts of the operands as cuBLAS sees them
  const int64_t ar = k.ta ? k.k : k.m, ac = k.ta ? k.m : k.k;
  const int64_t br = k.tb ? k.n : k.k, bc = k.tb ? k.k : k.n;
  LT_CHECK(cublasLtMatrixLayoutCreate(&p.a, CUDA_R_16BF, ar, ac, k.lda), "layout A");
  LT_CHECK(cublasLtMatrixLayoutCreate(&p.b, CUDA_R_16BF, br, bc, k.ldb), "layout B");
  LT_CHECK(cublasLtMatrixLayoutCreate(&p.d, CUDA_R_16BF, k.m, k.n, k.ldd), "layout D");
  cublasLtMatmulPreference_t pref;
  LT_CHECK(cublasLtMatmulPreferenceCreate(&pref), "PreferenceCreate");
  LT_CHECK(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES,
                                                &ws_cap, sizeof(ws_cap)), "pref workspace");
  cublasLtMatmulHeuristicResult_t res[1];
  int found = 0;
  const cublasStatus_t hs = cublasLtMatmulAlgoGetHeuristic(h, p.desc, p.a, p.b, p.d, p.d, pref, 1,
                                                           res, &found);
  cublasLtMatmulPreferenceDestroy(pref);
  if (hs != CUBLAS_STATUS_SUCCESS || found < 1)
    return fail(HET_ECUDA, "het_lt_matmul: no cuBLASLt algorithm for epilogue %d "
                "(m=%lld n=%lld k=%lld, status %d)", k.epi, (long long)k.m, (long long)k.n,
                (long long)k.k, (int)hs);
  p.algo = res[0].algo;
  p.ws = res[0].workspaceSize;
  *out = p;
  return HET_OK;
}

}  // namespace

extern "C" {

int het_lt_matmul(int trans_a, int trans_b, int64_t m, int64_t n, int64_t k, const void* a,
                  int64_t lda, const void* b, int64_t ldb, void* d, int64_t ldd, int epilogue,
                  void* bias, void* aux, int64_t ldaux, void* workspace, int64_t workspace_bytes,
                  void* stream) {
  if (m <= 0 || n <= 0 || k <= 0 || !a || !b || !d || epilogue < HET_LT_NONE ||
      epilogue > HET_LT_BGRADB || workspace_bytes < 0 || (workspace_bytes > 0 && !workspace))
    return fail(HET_EARG, "het_lt_matmul: bad args");
  if (epilogue != HET_LT_NONE && !bias)
    return fail(HET_EARG, "het_lt_matmul: epilogue %d needs the bias / bias-gradient vector",
                epilogue);
  if ((epilogue == HET_LT_GELU_AUX_BIAS || epilogue == HET_LT_DGELU_BGRAD) &&
      (!aux || ldaux < m || ldaux % 8))
    return fail(HET_EARG, "het_lt_matmul: epilogue %d needs aux with ld >= m, ld %% 8 == 0",
                epilogue);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16)
    return fail(HET_ECUDA, "het_lt_matmul: no current device");
  Key key{trans_a, trans_b, epilogue, m, n, k, lda, ldb, ldd,
          (epilogue == HET_LT_GELU_AUX_BIAS || epilogue == HET_LT_DGELU_BGRAD) ? ldaux : 0, dev};
  Plan p;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_handle[dev]) LT_CHECK(cublasLtCreate(&g_handle[dev]), "cublasLtCreate");
    auto it = g_plans.find(key);
    if (it == g_plans.end()) {
      int rc = make_plan(key, g_handle[dev], static_cast<size_t>(workspace_bytes), &p);
      if (rc != HET_OK) return rc;
      g_plans.emplace(key, p);
    } else {
      p = it->second;
    }
  }
  if (p.ws > static_cast<size_t>(workspace_bytes))
    return fail(HET_EARG, "het_lt_matmul: plan needs %zu workspace bytes", p.ws);
  // per-call pointers on the cached descriptor (serialised: the descriptor is shared)
  std::lock_guard<std::mutex> lk(g_mu);
  if (epilogue != HET_LT_NONE)
    LT_CHECK(cublasLtMatmulDescSetAttribute(p.desc, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias,
                                            sizeof(bias)), "BIAS_POINTER");
  if (epilogue == HET_LT_GELU_AUX_BIAS || epilogue == HET_LT_DGELU_BGRAD)
    LT_CHECK(cublasLtMatmulDescSetAttribute(p.desc, CUBLASLT_MATMUL_DESC_EPILOGUE_AUX_POINTER,
                                            &aux, sizeof(aux)), "AUX_POINTER");
  const float alpha = 1.f, beta = 0.f;
  LT_CHECK(cublasLtMatmul(g_handle[dev], p.desc, &alpha, a, p.a, b, p.b, &beta, d, p.d, d, p.d,
                          &p.algo, workspace, p.ws, static_cast<cudaStream_t>(stream)),
           "cublasLtMatmul");
  return HET_OK;
}

}  // extern "C"

// Uneven all-gather / reduce-scatter of one FSDP unit over NCCL 2.28
// (NVLink 5 / NVSwitch), dispatched on the shape of the unit's shard vector
// (UnitShardPlan row, reference core.py:229-240, sharding.py:48-98):
//
//   even      (all counts == U/N, offsets j*U/N)  -> ncclAllGather / ncclReduceScatter
//   skewed    (single owner, or few owners)       -> per-owner ring ncclBroadcast /
//                                                    ncclReduce inside one group, so
//                                                    an owner's egress is ~S, not (N-1)S
//   baseline  (north_star (2))                    -> grouped ncclSend / ncclRecv
//
// The Eq. 1 weight is applied by the producer (het_accumulate scales every contribution by m_i/B),
// so the reduction is a plain fp32 SUM on the wire.
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <cstring>
#include <vector>

#include "hetstep.h"
#include "hetstep_internal.cuh"

using het::fail;

namespace {

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return HET_OK;
  return fail(HET_ENCCL, "%s: %s", what, ncclGetErrorString(r));
}

#define NCCL_TRY(call)                                   \
  do {                                                   \
    int _rc = nccl_check((call), #call);                 \
    if (_rc != HET_OK) return _rc;                       \
  } while (0)

struct GroupGuard {  // ncclGroupEnd on every exit path once started
  bool open = false;
  int start() {
    int rc = nccl_check(ncclGroupStart(), "ncclGroupStart");
    open = rc == HET_OK;
    return rc;
  }
  int end() {
    open = false;
    return nccl_check(ncclGroupEnd(), "ncclGroupEnd");
  }
  ~GroupGuard() {
    if (open) ncclGroupEnd();
  }
};

int validate(const int64_t* counts, const int64_t* offsets, int nranks, int rank,
             int64_t* unit_total) {
  if (!counts || !offsets || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(HET_EARG, "bad rank/nranks (%d/%d) or null shard table", rank, nranks);
  int64_t pos = 0;
  for (int j = 0; j < nranks; ++j) {
    if (counts[j] < 0 || offsets[j] != pos)
      return fail(HET_EARG, "shard table not contiguous at rank %d (offset %lld, expected %lld)",
                  j, (long long)offsets[j], (long long)pos);
    pos += counts[j];
  }
  *unit_total = pos;
  return HET_OK;
}

bool is_even(const int64_t* counts, int nranks) {
  for (int j = 1; j < nranks; ++j)
    if (counts[j] != counts[0]) return false;
  return true;
}

ncclDataType_t nccl_dtype(int dtype) { return dtype == HET_DT_BF16 ? ncclBfloat16 : ncclFloat32; }

size_t dtype_size(int dtype) { return dtype == HET_DT_BF16 ? 2 : 4; }

}  // namespace

extern "C" {

int het_comm_unique_id(uint8_t out_id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  if (!out_id) return fail(HET_EARG, "het_comm_unique_id: null");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(out_id, &id, sizeof(id));
  return HET_OK;
}

int het_comm_init(void** comm_out, const uint8_t id[128], int nranks, int rank) {
  if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(HET_EARG, "het_comm_init: bad args");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm = nullptr;
  NCCL_TRY(ncclCommInitRank(&comm, nranks, uid, rank));
  *comm_out = comm;
  return HET_OK;
}

int het_comm_destroy(void* comm) {
  if (!comm) return HET_OK;
  NCCL_TRY(ncclCommDestroy(static_cast<ncclComm_t>(comm)));
  return HET_OK;
}

int het_allgather_uneven(const void* send, void* unit, const int64_t* counts,
                         const int64_t* offsets, int nranks, int rank, int dtype, int algo,
                         void* comm, void* stream) {
  int64_t total = 0;
  int rc = validate(counts, offsets, nranks, rank, &total);
  if (rc != HET_OK) return rc;
  if (dtype != HET_DT_BF16 && dtype != HET_DT_F32) return fail(HET_EARG, "bad dtype %d", dtype);
  if (!unit || (counts[rank] > 0 && !send)) return fail(HET_EARG, "null buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t es = dtype_size(dtype);
  char* dst = static_cast<char*>(unit);
  if (nranks == 1) {
    if (counts[0] && send != unit &&
        cudaMemcpyAsync(dst, send, counts[0] * es, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return het::check_launch("het_allgather_uneven(copy)");
    return HET_OK;
  }
  if (!comm) return fail(HET_EARG, "null communicator");
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  const ncclDataType_t dt = nccl_dtype(dtype);
  const bool even = is_even(counts, nranks);
  if (algo == HET_ALGO_EVEN && !even) return fail(HET_EARG, "HET_ALGO_EVEN on an uneven unit");
  if ((algo == HET_ALGO_AUTO || algo == HET_ALGO_EVEN) && even) {
    if (counts[0] == 0) return HET_OK;
    NCCL_TRY(ncclAllGather(send, unit, counts[0], dt, c, st));
    return HET_OK;
  }
  GroupGuard g;
  if ((rc = g.start()) != HET_OK) return rc;
  if (algo == HET_ALGO_P2P) {
    if (counts[rank] > 0 && send != dst + offsets[rank] * es &&
        cudaMemcpyAsync(dst + offsets[rank] * es, send, counts[rank] * es,
                        cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return het::check_launch("het_allgather_uneven(self)");
    for (int j = 0; j < nranks; ++j) {
      if (j == rank) continue;
      if (counts[rank] > 0) NCCL_TRY(ncclSend(send, counts[rank], dt, j, c, st));
      if (counts[j] > 0) NCCL_TRY(ncclRecv(dst + offsets[j] * es, counts[j], dt, j, c, st));
    }
  } else {  // per-owner pipelined ring broadcasts
    for (int j = 0; j < nranks; ++j) {
      if (counts[j] == 0) continue;
      const void* sb = (j == rank) ? send : static_cast<const void*>(dst + offsets[j] * es);
      NCCL_TRY(ncclBroadcast(sb, dst + offsets[j] * es, counts[j], dt, j, c, st));
    }
  }
  return g.end();
}

int het_reduce_scatter_uneven(const float* src, float* shard_out, const int64_t* counts,
                              const int64_t* offsets, int nranks, int rank, int algo,
                              void* comm, void* stream) {
  int64_t total = 0;
  int rc = validate(counts, offsets, nranks, rank, &total);
  if (rc != HET_OK) return rc;
  if (!src || (counts[rank] > 0 && !shard_out)) return fail(HET_EARG, "null buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (nranks == 1) {
    if (counts[0] && src != shard_out &&
        cudaMemcpyAsync(shard_out, src, counts[0] * sizeof(float), cudaMemcpyDeviceToDevice,
                        st) != cudaSuccess)
      return het::check_launch("het_reduce_scatter_uneven(copy)");
    return HET_OK;
  }
  if (!comm) return fail(HET_EARG, "null communicator");
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  const bool even = is_even(counts, nranks);
  if (algo == HET_ALGO_EVEN && !even) return fail(HET_EARG, "HET_ALGO_EVEN on an uneven unit");
  if ((algo == HET_ALGO_AUTO || algo == HET_ALGO_EVEN) && even) {
    if (counts[0] == 0) return HET_OK;
    NCCL_TRY(ncclReduceScatter(src, shard_out, counts[0], ncclFloat32, ncclSum, c, st));
    return HET_OK;
  }
  if (algo == HET_ALGO_P2P) {
    // a send/recv reduce-scatter needs N-1 staging slices on the owner; the
    // per-owner ring reduce below moves the same bytes without them
    return fail(HET_EARG, "HET_ALGO_P2P reduce-scatter is not provided; use "
                          "HET_ALGO_OWNER or HET_ALGO_AUTO");
  }
  GroupGuard g;
  if ((rc = g.start()) != HET_OK) return rc;
  for (int j = 0; j < nranks; ++j) {
    if (counts[j] == 0) continue;
    // recvbuff is only read on the root; non-roots pass their own slice
    float* rb = (j == rank) ? shard_out : const_cast<float*>(src + offsets[j]);
    NCCL_TRY(ncclReduce(src + offsets[j], rb, counts[j], ncclFloat32, ncclSum, j, c, st));
  }
  return g.end();
}

}  // extern "C"

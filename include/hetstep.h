/*
 * hetstep.h — C-ABI of the B200-native Cephalo uneven-FSDP train step.
 *
 * The reference (`hetplan`, /root/reference/pkg/src/hetplan) is pure Python and
 * has no FFI; its trainer exists only as the contract feeding it (planner
 * output, unit shards/offsets), the Eq. 1 math and the schedule. Each entry
 * point below implements one piece of that contract on sm_100a and cites what
 * it replaces. All calls are asynchronous and stream-ordered on the caller's
 * CUDA stream; buffers are owned by the caller (torch caching allocator);
 * nothing here allocates device memory except NCCL's own communicator state.
 *
 * Return codes: HET_OK, HET_EARG (bad sizes/pointers/alignment → Python
 * InputError), HET_ECUDA / HET_ENCCL (→ RuntimeError with het_last_error()).
 */
#ifndef HETSTEP_H_
#define HETSTEP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HET_OK 0
#define HET_EARG 1
#define HET_ECUDA 2
#define HET_ENCCL 3

#define HET_MAX_SEGS 256   /* segments per het_accumulate launch (kernel parameter table) */

/* One gradient tensor landing in a unit-sized fp32 accumulator. */
typedef struct {
  const void* src;    /* bf16 gradient, contiguous, n elements */
  int64_t dst_off;    /* element offset inside the unit accumulator */
  int64_t n;          /* elements */
} het_seg_t;

/* Accumulate modes (layered gradient accumulation, PAPER.md:653-660;
 * schedule sim.py:278-322: all l_i microbatches of a unit, then one RS).
 * Every contribution is pre-scaled by the rank's Eq. 1 weight w = m_i / B
 * (gradcheck.py:30-46), so acc ends as sum_k w*g_k and the reduce-scatter is
 * a plain SUM; with l_i == 1 the FIRST pass is the bf16->fp32 scale-cast. */
#define HET_ACC_ADD 0   /* acc += w*g  (microbatches 1..l_i-1, or a zeroed acc) */
#define HET_ACC_FIRST 1 /* acc  = w*g  (microbatch 0: no read of acc)           */

/* Library identity: returns a static string "hetstep <version> sm_100a". */
const char* het_version(void);
/* Thread-local text of the last non-OK return. */
const char* het_last_error(void);

/* ---- kernels --------------------------------------------------------- */

/* (1) pack: fp32 master shard -> bf16 all-gather send buffer, RNE.
 * Replaces: FSDP shard->flat-param cast before unshard;
 * the layout is sharding.py:89-95 offsets. 6 B/param. */
int het_pack_bf16(const float* src, void* dst_bf16, int64_t n, void* stream);

/* (4) layered accumulate-and-release over a segment table (one entry per
 * parameter gradient of a unit) into the unit's fp32 accumulator:
 * acc[dst_off + e] (=|+=) scale * bf16(src[e]). scale = m_i / B.
 * 6 B/param for HET_ACC_FIRST, 10 B/param for HET_ACC_ADD. The caller drops
 * its reference to the bf16 gradients after the call (release). */
int het_accumulate(float* acc, const het_seg_t* segs, int nseg, int mode, float scale,
                   void* stream);

/* (4') layered accumulate of nsrc consecutive microbatches in one pass:
 * segs is [nsrc][nseg] (source j of segment s at segs[j*nseg + s]; every
 * source of a segment has the same dst_off and n). Per element, in registers:
 * a = (FIRST ? scale*g_0 : fma(scale, g_0, acc)); a = fma(scale, g_j, a) for
 * j = 1..nsrc-1; acc = a — bit-identical to nsrc het_accumulate calls, with
 * one read and one write of acc instead of nsrc (2*nsrc+4 B/param FIRST,
 * 2*nsrc+8 ADD). 1 <= nsrc <= HET_MAX_ACC_SRC. */
#define HET_MAX_ACC_SRC 4
int het_accumulate_multi(float* acc, const het_seg_t* segs, int nseg, int nsrc, int mode,
                         float scale, void* stream);

/* (5) sharded AdamW over one rank's flat local shard (torch.optim.AdamW
 * formula, decoupled weight decay). Optional bf16 shadow write (the next
 * step's all-gather send buffer; fuses kernel (1)). 28 B/param, 30 with
 * shadow. step >= 1. Hyper-parameters are doubles: the fp32 coefficients
 * (1-b1, 1-b2, lr/(1-b1^t), ...) are derived in double exactly as torch
 * derives them from Python floats. Replaces: the paper's per-GPU Adam on the FSDP shard
 * (core.py:151-154 "16 B/param"). */
int het_adamw(float* p, const float* g, float* m, float* v, void* p_bf16_or_null, int64_t n,
              double lr, double beta1, double beta2, double eps, double weight_decay,
              int64_t step, void* stream);

/* The 7 fp32 AdamW coefficients het_adamw derives (in double, as torch) for
 * one step: {1-lr*wd, 1-b1, b2, 1-b2, sqrt(1-b2^t), eps, -lr/(1-b1^t)}. */
int het_adamw_coef(double lr, double beta1, double beta2, double eps, double weight_decay,
                   int64_t step, float* out7);
/* het_adamw with the coefficients read from device memory (coef7_dev, as
 * het_adamw_coef writes them) instead of kernel arguments: a CUDA graph of the
 * step replays it unchanged while the host refreshes the 28 bytes per step. */
int het_adamw_devcoef(float* p, const float* g, float* m, float* v, void* p_bf16_or_null,
                      int64_t n, const float* coef7_dev, void* stream);

/* (4b) embedding backward fused with layered accumulation of the root unit:
 *   acc[wte_off + t*d + c] += scale * sum_{i : token[i] == t} dy[i, c]
 *   acc[wpe_off + s*d + c] += scale * sum_{i : i % seq == s} dy[i, c]   (wpe_off >= 0)
 * dy: bf16 [rows, d] (rows = m*seq) upstream gradient of the embedding output.
 * order/seg_start/seg_token: the rows sorted by token id (stable) and the
 * run boundaries (nseg unique tokens), built on the device by the caller.
 * One CTA owns each token row / position row and sums its contributions in
 * fp32 in a fixed order: deterministic, no atomics, and no [vocab, d] bf16
 * dense gradient is ever materialised (replaces embedding_dense_backward +
 * het_accumulate of its output). */
int het_embedding_grad(float* acc, int64_t wte_off, int64_t wpe_off, const void* dy_bf16,
                       int64_t rows, int64_t d, const int32_t* order, const int32_t* seg_start,
                       const int32_t* seg_token, int64_t nseg, int64_t seq, float scale,
                       void* stream);

/* (4b') the same without a host round trip (CUDA-graph capturable): the run
 * count stays on the device (*nseg_dev), rows bounds it (one CTA per possible
 * run; CTAs past the live count exit), and sorted_tok is the stably sorted
 * token array, read at each run's start seg_start[b]. */
int het_embedding_grad_dev(float* acc, int64_t wte_off, int64_t wpe_off, const void* dy_bf16,
                           int64_t rows, int64_t d, const int32_t* order,
                           const int32_t* seg_start, const int32_t* sorted_tok,
                           const int32_t* nseg_dev, int64_t seq, float scale, void* stream);

/* Fused LayerNorm of the transformer units (bf16 activations, fp32 stats),
 * d in {256, 768, 1024}. Forward writes y, per-row mean and rstd; backward
 * writes dx and dgamma/dbeta (bf16) using `partial`, a caller-owned fp32
 * scratch of het_layernorm_partial_floats(d) floats. Deterministic. */
int64_t het_layernorm_partial_floats(int64_t d);
int het_layernorm_fwd(const void* x, const void* w, const void* b, void* y, float* mean,
                      float* rstd, int64_t rows, int64_t d, float eps, void* stream);
int het_layernorm_bwd(const void* dy, const void* x, const void* w, const float* mean,
                      const float* rstd, void* dx, void* dgamma, void* dbeta, float* partial,
                      int64_t rows, int64_t d, void* stream);

/* Fused next-token cross-entropy over bf16 logits [rows, vocab] (vocab % 8 == 0):
 * forward writes per-row log-sum-exp and loss; backward writes
 * dlogits = (*grad_loss / rows) * (softmax - onehot(target)), grad_loss being
 * the device-resident upstream gradient of the mean loss (no host sync);
 * dlogits may alias logits. */
int het_xent_fwd(const void* logits, const int64_t* target, int64_t rows, int64_t vocab,
                 float* lse, float* loss, void* stream);
int het_xent_bwd(const void* logits, const int64_t* target, int64_t rows, int64_t vocab,
                 const float* lse, const float* grad_loss, void* dlogits, void* stream);

/* Fused RMSNorm (Llama units), d in {256, 768, 1024, 2048}; same conventions
 * as the LayerNorm pair (partial scratch of het_rmsnorm_partial_floats(d)). */
int64_t het_rmsnorm_partial_floats(int64_t d);
int het_rmsnorm_fwd(const void* x, const void* w, void* y, float* rstd, int64_t rows, int64_t d,
                    float eps, void* stream);
int het_rmsnorm_bwd(const void* dy, const void* x, const void* w, const float* rstd, void* dx,
                    void* dgamma, float* partial, int64_t rows, int64_t d, void* stream);
/* Rotary position embedding in place on bf16 [rows, heads, dh] (row r at
 * position r % seq, rotate-half pairs); inverse=1 applies the backward
 * (inverse) rotation. */
/* Residual add fused into the norms: xsum = bf16(x + r) is written and
 * normalised (forward); the backward adds the residual path's gradient dres
 * to the norm's input gradient in the same pass (dres may be NULL). */
int het_layernorm_add_fwd(const void* x, const void* r, const void* w, const void* b, void* xsum,
                          void* y, float* mean, float* rstd, int64_t rows, int64_t d, float eps,
                          void* stream);
int het_layernorm_bwd_add(const void* dy, const void* dres, const void* x, const void* w,
                          const float* mean, const float* rstd, void* dx, void* dgamma, void* dbeta,
                          float* partial, int64_t rows, int64_t d, void* stream);
int het_rmsnorm_add_fwd(const void* x, const void* r, const void* w, void* xsum, void* y,
                        float* rstd, int64_t rows, int64_t d, float eps, void* stream);
int het_rmsnorm_bwd_add(const void* dy, const void* dres, const void* x, const void* w,
                        const float* rstd, void* dx, void* dgamma, float* partial, int64_t rows,
                        int64_t d, void* stream);

int het_rope_inplace(void* x, int64_t rows, int heads, int dh, int64_t seq, int inverse,
                     void* stream);

/* Fused q/k/v projection output [rows, 3*heads*dh] (q | k | v per row) ->
 * rotary-embedded q and k and a copy of v, each contiguous [rows, heads, dh]
 * (row r at position r % seq); merge = the backward: dq, dk (inverse
 * rotation) and dv into one [rows, 3*heads*dh] gradient. dh % 16 == 0. */
int het_rope_qkv_split(const void* qkv, void* q, void* k, void* v, int64_t rows, int heads, int dh,
                       int64_t seq, void* stream);
int het_rope_qkv_merge(const void* dq, const void* dk, const void* dv, void* dqkv, int64_t rows,
                       int heads, int dh, int64_t seq, void* stream);

/* SwiGLU on bf16: out[r, j] = silu(a[r, j]) * b[r, j] for r < rows, j < f,
 * a and b with row stride ld (separate tensors, or the two halves of one
 * [rows, 2f] projection), out contiguous [rows, f]. Rounds like torch's
 * F.silu(a) * b (silu to bf16, then the product). Backward: da, db (row
 * stride ldg) from dout [rows, f]. */
int het_swiglu_fwd(const void* a, const void* b, int64_t ld, void* out, int64_t rows, int64_t f,
                   void* stream);
int het_swiglu_bwd(const void* dout, const void* a, const void* b, int64_t ld, void* da, void* db,
                   int64_t ldg, int64_t rows, int64_t f, void* stream);

/* Linear-layer epilogues (GPT/BERT units), bf16 in/out with fp32 sums:
 * het_bias_grad:     db[c] = sum_r g[r, c] over a row-major [rows, n] gradient
 *                    (deterministic two-pass column sum; `partial` holds
 *                    het_colsum_partial_floats(rows, n) floats of scratch);
 * het_gelu_fwd:      y = tanh-approximate GELU(x) over n elements;
 * het_gelu_bwd_bias: dpre = GELU'(pre) * dy and db = column sums of dpre
 *                    in one pass (the bias gradient of the projection that
 *                    produced `pre`). */
int64_t het_colsum_partial_floats(int64_t rows, int64_t n);
int het_bias_grad(const void* g, int64_t rows, int64_t n, void* db, float* partial, void* stream);
int het_gelu_fwd(const void* x, void* y, int64_t n, void* stream);
int het_gelu_bwd_bias(const void* dy, const void* pre, void* dpre, int64_t rows, int64_t n,
                      void* db, float* partial, void* stream);

/* Launch-shape tuning knobs (process-wide; defaults are the measured best).
 * HET_TUNE_ACC_VARIANT: het_accumulate CTA shape index 0..5
  * ((threads, loads in flight) = (256,4) (256,2) (256,1) (512,2) (512,1) (128,4));
 * default 4, measured fastest on B200 (tools/acc_bench.cu). */
#define HET_TUNE_ACC_VARIANT 1
/* HET_TUNE_SM_BUDGET: SMs the persistent grids (accumulate, AdamW, pack, fill)
 * are sized for: a rank whose compute stream lives in a green-context
 * partition of nsm SMs sets nsm, so one wave fills its partition instead of
 * 148 x k CTAs queueing behind it. 0 = the whole device (default). */
#define HET_TUNE_SM_BUDGET 2
/* HET_TUNE_SYMM_TIMEOUT_MS: spin limit of the fused collectives' cross-rank
 * barriers (default 10000 ms); after it the kernel records HET_SYMM_TIMEOUT. */
#define HET_TUNE_SYMM_TIMEOUT_MS 3
/* HET_TUNE_ACC_GRID: grid of the accumulate kernels. 0 = persistent (one wave
 * of the CTAs resident on the rank's SMs, each walking its share of chunks);
 * 1 = one CTA per chunk, so the hardware scheduler spreads the work over
 * whatever SMs are free (a persistent wave whose SMs are partly held by the
 * fused collectives' CTAs runs as two waves). */
#define HET_TUNE_ACC_GRID 4
int het_tune(int key, int value);

/* Emulation diagnostic: `ctas` CTAs each write the %smid they ran on to
 * out[blockIdx]; launched on a green-context stream, the distinct values are
 * the SMs of its partition (tests/test_emulation_gpu.py). */
int het_probe_smid(int32_t* out, int ctas, void* stream);

/* fill / zero helpers used by the step driver (idle ranks, pads) */
int het_fill_f32(float* dst, float value, int64_t n, void* stream);

/* ---- collectives (NCCL 2.28 over NVLink 5 / NVSwitch) ----------------- */

/* 128-byte NCCL unique id produced on rank 0 and broadcast by the host. */
int het_comm_unique_id(uint8_t out_id[128]);
int het_comm_init(void** comm_out, const uint8_t id[128], int nranks, int rank);
int het_comm_destroy(void* comm);

#define HET_DT_BF16 0
#define HET_DT_F32 1

#define HET_ALGO_AUTO 0      /* even -> AllGather/ReduceScatter, else per-owner */
#define HET_ALGO_P2P 1       /* grouped ncclSend/ncclRecv (north_star baseline)  */
#define HET_ALGO_OWNER 2     /* grouped per-owner ncclBroadcast / ncclReduce     */
#define HET_ALGO_EVEN 3      /* require even: ncclAllGather / ncclReduceScatter  */

/* (2) uneven all-gather of one unit: rank j contributes counts[j] elements
 * from `send` into unit[offsets[j] : offsets[j]+counts[j]] on every rank.
 * counts/offsets are host arrays of length nranks (UnitShardPlan row,
 * core.py:229-240). Replaces FSDP's generalized AllGather
 * (PAPER.md:549, 648-651); schedule sim.py:344-363. */
int het_allgather_uneven(const void* send, void* unit, const int64_t* counts,
                         const int64_t* offsets, int nranks, int rank, int dtype, int algo,
                         void* comm, void* stream);

/* (3) uneven reduce-scatter of a unit: shard_out[0:counts[rank]] =
 * sum_j src_j[offsets[rank] : +counts[rank]] where every rank's src was
 * pre-scaled by its Eq. 1 weight in het_accumulate. fp32 in, fp32 out.
 * Replaces FSDP's generalized ReduceScatter + Cephalo's reweighting
 * (gradcheck.py:30-46); issue point sim.py:364-368. */
int het_reduce_scatter_uneven(const float* src, float* shard_out, const int64_t* counts,
                              const int64_t* offsets, int nranks, int rank, int algo,
                              void* comm, void* stream);

/* ---- fused collectives on a symmetric buffer (NVLS multicast / peer) ---- */

#define HET_MAX_RANKS 8
#define HET_SYMM_MAX_CTAS 256
#define HET_SYMM_CHANNELS 2   /* independent barrier channels: 0 = AG stream, 1 = RS stream */
#define HET_SYMM_TIMEOUT 17   /* het_symm_status(): a cross-rank barrier timed out */

/* Route policy of the fused collectives. AUTO picks per call from the shard
 * vector: NVLS multicast moves S bytes over every GPU's link, peer push/pull
 * moves max((N-1) max_j s_j, S - min_i s_i); the cheaper one runs. */
#define HET_SYMM_AUTO 0
#define HET_SYMM_MULTICAST 1
#define HET_SYMM_PEER 2
/* All-gather only (the reduce-scatter treats it as AUTO): peer push where
 * each big owner hands a share of its range to a small owner, which forwards
 * it, balancing link egress on skewed shard vectors (N >= 3). */
#define HET_SYMM_RELAY 3
/* All-gather and both reduce-scatters: heavy owners hand pieces of their range
 * to light ranks ("helpers"). AG: the owner pushes a piece to its helper only
 * and the helper forwards it to the other N-2 ranks. RS: the helper reduces
 * the piece over all ranks into a staging copy in its own buffer and the owner
 * pulls the reduced piece. Pieces stream in grid-stride iterations with
 * CTA-pairwise progress flags, so forwarding / pulling overlaps production.
 * A single owner then moves S (not (N-1) S) over its link; the plan
 * (het_symm_helper_plan) balances every link's load. N >= 3. */
#define HET_SYMM_HELPERS 4
/* fp32 reduce-scatter only (others treat it as HELPERS; without a multicast
 * object it is HELPERS): the helpers, and the owner for its direct part, reduce
 * through the switch (multimem.ld_reduce: 4 B per element in) instead of
 * pulling N-1 peer ranges, and the owner pulls the staged sums. Not rank-ordered
 * (like HET_SYMM_MULTICAST). */
#define HET_SYMM_HELPERS_MC 5

/* Ops of het_symm_helper_plan */
#define HET_OP_AG 0
#define HET_OP_RS 1
#define HET_OP_RS_BF16 2
#define HET_OP_RS_MC 3     /* fp32 RS under HET_SYMM_HELPERS_MC (its link costs) */

/* A buffer allocated at the same byte layout on every rank (torch symmetric
 * memory is the plumbing): peer_base[j] = its address on rank j mapped into
 * this process (UVA peer mapping), mc_base = NVLS multicast address or 0.
 * signal_off = byte offset of a zeroed area of het_symm_signal_bytes(). */
typedef struct {
  int32_t nranks;
  int32_t rank;
  uint64_t peer_base[HET_MAX_RANKS];
  uint64_t mc_base;
  uint64_t signal_off;
} het_symm_t;

int64_t het_symm_signal_bytes(void);
/* Test support: all N ranks of one fused collective (op = HET_OP_AG / RS /
 * RS_BF16 with the given policy) as ONE cooperative launch on one GPU, CTA b of
 * rank r at blockIdx r * ctas + b, descs[r] being rank r's descriptor over one
 * allocation (mc_base = 0). The same kernel bodies and barriers as N real
 * launches with every CTA co-resident by construction (refused with HET_EARG
 * if N * ctas CTAs cannot be). srcs[r] / outs[r]: rank r's fp32 range (AG) or
 * output shard (RS). Synchronous. */
int het_symm_virtual(int op, int nranks, const het_symm_t* descs, const float* const* srcs,
                     float* const* outs, const int64_t* counts, const int64_t* offsets,
                     uint64_t off, const float* weights, uint32_t epoch, int channel,
                     int end_barrier, int policy, uint64_t stage_off, int ctas, void* stream);

/* Sticky device status of the symmetric kernels (0 or HET_SYMM_TIMEOUT).
 * Synchronous (device-wide copy); reset=1 clears it. */
int het_symm_status(int reset);
/* The same status written to *dst by a one-thread kernel on `stream`, after
 * everything queued before it: dst may be pinned host memory (device-mapped
 * under UVA), so the step driver checks it from an event, without a device
 * sync, and raises instead of training on unsynchronised gradients. */
int het_symm_status_async(int32_t* dst, void* stream);

/* Device-resident barrier epochs, for a CUDA graph that replays a multi-rank
 * step (no host counter can change inside a replay). An epoch argument with
 * HET_SYMM_EPOCH_DEVICE set means base[channel] + (epoch & ~FLAG), base being
 * a counter in this rank's signal area (after the barrier slots, inside
 * het_symm_signal_bytes()). het_symm_epoch_set seeds it (from the host
 * counter, before capture); het_symm_epoch_add(delta = the channel's launches
 * per step), queued after the step's last collective of that channel and
 * captured with it, advances it every replay. Both are one-thread kernels on
 * `stream`. Every rank issues the same epoch sequence whether it replays a
 * graph or runs eagerly with host epochs. */
#define HET_SYMM_EPOCH_DEVICE 0x80000000u
int het_symm_epoch_set(const het_symm_t* s, int channel, uint32_t value, void* stream);
int het_symm_epoch_add(const het_symm_t* s, int channel, uint32_t delta, void* stream);

/* (1)+(2) fused: rank r rounds its fp32 master range src[0:counts[r]] to bf16
 * and stores it at unit_off + 2*offsets[r] on EVERY rank with one multicast
 * store (NVLS) or per-peer stores. In-kernel start/end barriers; `epoch`
 * must increase by one per call on `channel` on every rank. */
int het_symm_allgather_pack(const het_symm_t* s, const float* src, uint64_t unit_off,
                            const int64_t* counts, const int64_t* offsets, uint32_t epoch,
                            int channel, int policy, int ctas, void* stream);

/* (3) fused: out[0:counts[r]] = sum_j acc_j[offsets[r] : +counts[r]] where
 * acc_j is the fp32 accumulator at acc_off on rank j (already Eq. 1-scaled),
 * summed in the switch by multimem.ld_reduce (or peer loads). end_barrier=1
 * additionally waits until every rank finished reading this rank's acc. */
int het_symm_reduce_scatter(const het_symm_t* s, uint64_t acc_off, float* out,
                            const int64_t* counts, const int64_t* offsets, uint32_t epoch,
                            int channel, int end_barrier, int policy, int ctas, void* stream);

/* (3) fused, bf16 wire: out[0:counts[r]] = sum_j weights[j] * grad_j[offsets[r] : +counts[r]]
 * in fp32, where grad_j is rank j's UNSCALED bf16 unit gradient at grad_off
 * (l_j = 1: the microbatch gradient itself) and weights[j] = m_j / B (Eq. 1).
 * The per-rank weighting and the bf16 -> fp32 cast happen inside the
 * reduce-scatter; half the link bytes of the fp32 form. Peer loads, summed
 * in rank order (so equal, bit for bit, to het_symm_reduce_scatter's peer
 * route over pre-scaled fp32 accumulators). */
int het_symm_reduce_scatter_bf16(const het_symm_t* s, uint64_t grad_off, float* out,
                                 const int64_t* counts, const int64_t* offsets,
                                 const float* weights, uint32_t epoch, int channel,
                                 int end_barrier, int policy, uint64_t stage_off, int ctas,
                                 void* stream);
/* policy: HET_SYMM_AUTO / HET_SYMM_PEER (peer pull) or HET_SYMM_HELPERS, whose
 * helpers write fp32 partial results at stage_off (an fp32 unit-sized region of
 * the symmetric buffer, 16-byte aligned; unused otherwise). The helper routes
 * always end with the cross-rank barrier (owners have read the staging). */

/* The helper plan the kernels use for `op` (HET_OP_*) on this shard table:
 * direct body vectors per rank (out_direct[nranks]), (owner, helper) pairs of
 * the pieces (out_pieces[2 * max_pieces]) and the per-rank link load in bytes
 * (link_load[nranks]: AG egress, RS ingress). Host only. Returns the number
 * of pieces, or -HET_EARG. */
int het_symm_helper_plan(int op, int nranks, const int64_t* counts, const int64_t* offsets,
                         uint64_t off, int64_t* out_direct, int32_t* out_pieces, int max_pieces,
                         double* link_load);

/* bf16 gradient segments copied (unscaled) into one bf16 unit buffer:
 * dst[segs[i].dst_off : +n] = segs[i].src. The l_i = 1 staging of the bf16-wire
 * reduce-scatter (4 B/param instead of the fp32 accumulate's 6). */
int het_gather_bf16(void* dst, const het_seg_t* segs, int nseg, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HETSTEP_H_ */

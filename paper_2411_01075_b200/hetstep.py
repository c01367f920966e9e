"""ctypes binding of the sm_100a C-ABI (``include/hetstep.h``).

Every function takes torch CUDA tensors, checks dtype/contiguity/device, and
launches on the caller's current CUDA stream (or an explicit one). There is
no CPU or PyTorch fallback: if ``libhetstep.so`` cannot be loaded, or a tensor
is not on a CUDA device, the call raises.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import torch

from ._build import STEP_LIB, build_step
from .core import InputError

HET_OK, HET_EARG, HET_ECUDA, HET_ENCCL = 0, 1, 2, 3
HET_MAX_SEGS = 256
ACC_ADD, ACC_FIRST = 0, 1
DT_BF16, DT_F32 = 0, 1
ALGO_AUTO, ALGO_P2P, ALGO_OWNER, ALGO_EVEN = 0, 1, 2, 3
ALGO_SYMM = 4            # fused kernels on a symmetric buffer (NVLS multicast / peer)
HET_MAX_RANKS = 8
HET_SYMM_MAX_CTAS = 256
HET_SYMM_TIMEOUT = 17
SYMM_AUTO, SYMM_MULTICAST, SYMM_PEER, SYMM_RELAY, SYMM_HELPERS = 0, 1, 2, 3, 4
SYMM_HELPERS_MC = 5              # fp32 RS: helpers reduce in the switch (multimem.ld_reduce)
SYMM_CHANNELS = 2                # HET_SYMM_CHANNELS: 0 = AG stream, 1 = RS stream
EPOCH_DEVICE = 0x80000000        # HET_SYMM_EPOCH_DEVICE
OP_AG, OP_RS, OP_RS_BF16, OP_RS_MC = 0, 1, 2, 3

EXPORTS = ("het_version", "het_last_error", "het_pack_bf16", "het_accumulate", "het_adamw",
           "het_fill_f32", "het_tune", "het_embedding_grad", "het_layernorm_partial_floats",
           "het_layernorm_fwd", "het_layernorm_bwd", "het_xent_fwd", "het_xent_bwd",
           "het_rmsnorm_partial_floats", "het_rmsnorm_fwd", "het_rmsnorm_bwd", "het_rope_inplace",
           "het_swiglu_fwd", "het_swiglu_bwd", "het_rope_qkv_split", "het_rope_qkv_merge",
           "het_layernorm_add_fwd", "het_layernorm_bwd_add", "het_rmsnorm_add_fwd",
           "het_rmsnorm_bwd_add", "het_colsum_partial_floats", "het_bias_grad",
           "het_gelu_fwd", "het_gelu_bwd_bias", "het_comm_unique_id", "het_comm_init", "het_comm_destroy",
           "het_allgather_uneven", "het_reduce_scatter_uneven", "het_symm_signal_bytes",
           "het_symm_status", "het_symm_allgather_pack", "het_symm_reduce_scatter",
           "het_symm_reduce_scatter_bf16", "het_gather_bf16", "het_accumulate_multi",
           "het_embedding_grad_dev", "het_adamw_coef", "het_adamw_devcoef",
           "het_symm_status_async", "het_symm_epoch_set", "het_symm_epoch_add", "het_probe_smid", "het_symm_helper_plan",
           "het_symm_virtual")


class HetSeg(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("dst_off", ctypes.c_int64), ("n", ctypes.c_int64)]


class HetSymm(ctypes.Structure):
    _fields_ = [("nranks", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("peer_base", ctypes.c_uint64 * HET_MAX_RANKS), ("mc_base", ctypes.c_uint64),
                ("signal_off", ctypes.c_uint64)]


_lib: ctypes.CDLL | None = None


def load(build: bool = False) -> ctypes.CDLL:
    """Load (optionally building first) the in-tree libhetstep.so."""
    global _lib
    if _lib is not None:
        return _lib
    if build or not STEP_LIB.exists():
        build_step()
    lib = ctypes.CDLL(str(STEP_LIB))
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    f32, f64 = ctypes.c_float, ctypes.c_double
    sig = {
        "het_version": ([], ctypes.c_char_p),
        "het_last_error": ([], ctypes.c_char_p),
        "het_pack_bf16": ([vp, vp, i64, vp], i32),
        "het_accumulate": ([vp, ctypes.POINTER(HetSeg), i32, i32, f32, vp], i32),
        "het_accumulate_multi": ([vp, ctypes.POINTER(HetSeg), i32, i32, i32, f32, vp], i32),
        "het_adamw": ([vp, vp, vp, vp, vp, i64, f64, f64, f64, f64, f64, i64, vp], i32),
        "het_adamw_coef": ([f64, f64, f64, f64, f64, i64, ctypes.POINTER(f32)], i32),
        "het_adamw_devcoef": ([vp, vp, vp, vp, vp, i64, vp, vp], i32),
        "het_fill_f32": ([vp, f32, i64, vp], i32),
        "het_tune": ([i32, i32], i32),
        "het_layernorm_partial_floats": ([i64], i64),
        "het_layernorm_fwd": ([vp, vp, vp, vp, vp, vp, i64, i64, f32, vp], i32),
        "het_layernorm_bwd": ([vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, vp], i32),
        "het_xent_fwd": ([vp, vp, i64, i64, vp, vp, vp], i32),
        "het_rmsnorm_partial_floats": ([i64], i64),
        "het_rmsnorm_fwd": ([vp, vp, vp, vp, i64, i64, f32, vp], i32),
        "het_rmsnorm_bwd": ([vp, vp, vp, vp, vp, vp, vp, i64, i64, vp], i32),
        "het_rope_inplace": ([vp, i64, i32, i32, i64, i32, vp], i32),
        "het_xent_bwd": ([vp, vp, i64, i64, vp, vp, vp, vp], i32),
        "het_swiglu_fwd": ([vp, vp, i64, vp, i64, i64, vp], i32),
        "het_rope_qkv_split": ([vp, vp, vp, vp, i64, i32, i32, i64, vp], i32),
        "het_layernorm_add_fwd": ([vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, f32, vp], i32),
        "het_layernorm_bwd_add": ([vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, vp], i32),
        "het_rmsnorm_add_fwd": ([vp, vp, vp, vp, vp, vp, i64, i64, f32, vp], i32),
        "het_rmsnorm_bwd_add": ([vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, vp], i32),
        "het_rope_qkv_merge": ([vp, vp, vp, vp, i64, i32, i32, i64, vp], i32),
        "het_colsum_partial_floats": ([i64, i64], i64),
        "het_bias_grad": ([vp, i64, i64, vp, vp, vp], i32),
        "het_gelu_fwd": ([vp, vp, i64, vp], i32),
        "het_gelu_bwd_bias": ([vp, vp, vp, i64, i64, vp, vp, vp], i32),
        "het_swiglu_bwd": ([vp, vp, vp, i64, vp, vp, i64, i64, i64, vp], i32),
        "het_embedding_grad": ([vp, i64, i64, vp, i64, i64, vp, vp, vp, i64, i64, f32, vp], i32),
        "het_embedding_grad_dev": ([vp, i64, i64, vp, i64, i64, vp, vp, vp, vp, i64, f32, vp],
                                   i32),
        "het_comm_unique_id": ([ctypes.c_char_p], i32),
        "het_comm_init": ([ctypes.POINTER(vp), ctypes.c_char_p, i32, i32], i32),
        "het_comm_destroy": ([vp], i32),
        "het_allgather_uneven": ([vp, vp, ctypes.POINTER(i64), ctypes.POINTER(i64), i32, i32, i32,
                                  i32, vp, vp], i32),
        "het_reduce_scatter_uneven": ([vp, vp, ctypes.POINTER(i64), ctypes.POINTER(i64), i32, i32,
                                       i32, vp, vp], i32),
        "het_symm_signal_bytes": ([], i64),
        "het_symm_status": ([i32], i32),
        "het_symm_status_async": ([vp, vp], i32),
        "het_symm_epoch_set": ([ctypes.POINTER(HetSymm), i32, ctypes.c_uint32, vp], i32),
        "het_symm_epoch_add": ([ctypes.POINTER(HetSymm), i32, ctypes.c_uint32, vp], i32),
        "het_probe_smid": ([vp, i32, vp], i32),
        "het_symm_allgather_pack": ([ctypes.POINTER(HetSymm), vp, ctypes.c_uint64,
                                     ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.c_uint32,
                                     i32, i32, i32, vp], i32),
        "het_symm_reduce_scatter": ([ctypes.POINTER(HetSymm), ctypes.c_uint64, vp,
                                     ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.c_uint32,
                                     i32, i32, i32, i32, vp], i32),
        "het_symm_reduce_scatter_bf16": ([ctypes.POINTER(HetSymm), ctypes.c_uint64, vp,
                                          ctypes.POINTER(i64), ctypes.POINTER(i64),
                                          ctypes.POINTER(f32), ctypes.c_uint32, i32, i32, i32,
                                          ctypes.c_uint64, i32, vp], i32),
        "het_symm_virtual": ([i32, i32, ctypes.POINTER(HetSymm), ctypes.POINTER(vp),
                              ctypes.POINTER(vp), ctypes.POINTER(i64), ctypes.POINTER(i64),
                              ctypes.c_uint64, ctypes.POINTER(f32), ctypes.c_uint32, i32, i32,
                              i32, ctypes.c_uint64, i32, vp], i32),
        "het_symm_helper_plan": ([i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                  ctypes.c_uint64, ctypes.POINTER(i64),
                                  ctypes.POINTER(ctypes.c_int32), i32,
                                  ctypes.POINTER(f64)], i32),
        "het_gather_bf16": ([vp, ctypes.POINTER(HetSeg), i32, vp], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def version() -> str:
    return load().het_version().decode()


LAUNCHES = 0      # owned kernel launches issued by this process (incl. model-side kernels)
_NOT_LAUNCHES = ("het_comm_unique_id", "het_comm_init", "het_comm_destroy", "het_tune",
                 "het_symm_helper_plan",
                 "het_symm_status", "het_allgather_uneven", "het_reduce_scatter_uneven",  # NCCL
                 "het_adamw_coef")                                                 # host-only


def _check(rc: int, what: str) -> None:
    global LAUNCHES
    if rc == HET_OK:
        if what not in _NOT_LAUNCHES:
            LAUNCHES += 1
        return
    msg = load().het_last_error().decode()
    if rc == HET_EARG:
        raise InputError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed ({'CUDA' if rc == HET_ECUDA else 'NCCL'}): {msg}")


def _cuda(t: torch.Tensor, dtype: torch.dtype, name: str) -> int:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InputError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise InputError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise InputError(f"{name} must be contiguous")
    return t.data_ptr()


def _stream(stream: torch.cuda.Stream | None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# Weight-gradient destinations. The step registers, for one unit's backward,
# where each parameter's bf16 gradient should land (its slot in the symmetric
# bf16-wire staging buffer); the fused autograd ops below write their weight /
# bias / norm gradients there directly, so no staging copy follows. Keyed by
# (data_ptr, shape) of the parameter tensor the op sees.
_GRAD_DST: dict[tuple[int, tuple[int, ...]], torch.Tensor] = {}


def _key(p: torch.Tensor) -> tuple:
    return (p.data_ptr(), tuple(p.shape), p.dtype, p.device)


def grad_out(p) -> torch.Tensor:
    """The registered destination of the gradient of p (a tensor or its _key),
    else a fresh tensor."""
    ptr, shape, dtype, device = p if isinstance(p, tuple) else _key(p)
    d = _GRAD_DST.get((ptr, shape))
    if d is not None and d.dtype == dtype:
        return d
    return torch.empty(shape, dtype=dtype, device=device)


class grad_destinations:
    """Context manager registering {(data_ptr, shape): destination} for a backward."""

    def __init__(self, mapping: dict):
        self.mapping = mapping

    def __enter__(self):
        _GRAD_DST.update(self.mapping)
        return self

    def __exit__(self, *exc):
        for k in self.mapping:
            _GRAD_DST.pop(k, None)


def pack_bf16(src: torch.Tensor, dst: torch.Tensor, stream=None) -> None:
    n = src.numel()
    if dst.numel() != n:
        raise InputError("pack_bf16: size mismatch")
    _check(load().het_pack_bf16(_cuda(src, torch.float32, "src"),
                                _cuda(dst, torch.bfloat16, "dst"), n, _stream(stream)),
           "het_pack_bf16")


def accumulate(acc: torch.Tensor, grads: Sequence[tuple[torch.Tensor, int]], first: bool,
               scale: float, stream=None, events=None) -> None:
    """acc[off:off+g.numel()] (=|+=) scale * g for every (g, off); g bf16.
    `events` = (start, end) CUDA events recorded right around the launch(es),
    after the host built the segment table (so a timer sees the kernel, not
    the host work)."""
    if not grads:
        return
    if len(grads) > HET_MAX_SEGS:
        parts = range(0, len(grads), HET_MAX_SEGS)
        for j, i in enumerate(parts):
            ev = None if events is None else (events[0] if j == 0 else None,
                                              events[1] if j == len(parts) - 1 else None)
            accumulate(acc, grads[i:i + HET_MAX_SEGS], first, scale, stream, ev)
        return
    cap = acc.numel()
    rows: list[list[int]] = []      # [src, dst_off, n]; back-to-back segments coalesce
    for i, (g, off) in enumerate(grads):
        if off < 0 or off + g.numel() > cap:
            raise InputError(f"accumulate: segment {i} [{off}, {off + g.numel()}) outside {cap}")
        src, n = _cuda(g, torch.bfloat16, f"grad[{i}]"), g.numel()
        if rows and rows[-1][0] + 2 * rows[-1][2] == src and rows[-1][1] + rows[-1][2] == off:
            rows[-1][2] += n
        else:
            rows.append([src, off, n])
    segs = (HetSeg * len(rows))()
    for i, (src, off, n) in enumerate(rows):
        segs[i].src, segs[i].dst_off, segs[i].n = src, off, n
    accp = _cuda(acc, torch.float32, "acc")
    if events is not None and events[0] is not None:
        events[0].record()
    _check(load().het_accumulate(accp, segs, len(rows), ACC_FIRST if first else ACC_ADD,
                                 float(scale), _stream(stream)), "het_accumulate")
    if events is not None and events[1] is not None:
        events[1].record()


HET_MAX_ACC_SRC = 4


def accumulate_multi(acc: torch.Tensor, sources: Sequence[Sequence[torch.Tensor]],
                     offsets: Sequence[int], first: bool, scale: float, stream=None,
                     events=None) -> None:
    """Layered accumulate of several consecutive microbatches in one pass:
    sources[j][s] is microbatch j's bf16 gradient of segment s, landing at
    acc[offsets[s]:]; acc (=|+=) scale*g_0, then += scale*g_j in order, in
    registers — bit-identical to len(sources) accumulate() calls with one
    read and one write of acc."""
    nsrc = len(sources)
    if nsrc == 0 or not offsets:
        return
    if nsrc > HET_MAX_ACC_SRC:
        raise InputError(f"accumulate_multi: at most {HET_MAX_ACC_SRC} sources, got {nsrc}")
    if any(len(src) != len(offsets) for src in sources):
        raise InputError("accumulate_multi: every source needs one tensor per offset")
    if len(offsets) > HET_MAX_SEGS:
        parts = range(0, len(offsets), HET_MAX_SEGS)
        for j, i in enumerate(parts):
            ev = None if events is None else (events[0] if j == 0 else None,
                                              events[1] if j == len(parts) - 1 else None)
            accumulate_multi(acc, [src[i:i + HET_MAX_SEGS] for src in sources],
                             offsets[i:i + HET_MAX_SEGS], first, scale, stream, ev)
        return
    cap = acc.numel()
    rows: list[list[int]] = []      # [dst_off, n, src_0, ..., src_{nsrc-1}]
    for i, off in enumerate(offsets):
        n = sources[0][i].numel()
        if off < 0 or off + n > cap:
            raise InputError(f"accumulate_multi: segment {i} [{off}, {off + n}) outside {cap}")
        ptrs = []
        for j, src in enumerate(sources):
            if src[i].numel() != n:
                raise InputError(f"accumulate_multi: source {j} segment {i} has "
                                 f"{src[i].numel()} elements, source 0 has {n}")
            ptrs.append(_cuda(src[i], torch.bfloat16, f"src[{j}][{i}]"))
        if rows and rows[-1][0] + rows[-1][1] == off and all(
                rows[-1][2 + j] + 2 * rows[-1][1] == ptrs[j] for j in range(nsrc)):
            rows[-1][1] += n        # back-to-back in the accumulator and in every source
        else:
            rows.append([off, n] + ptrs)
    segs = (HetSeg * (len(rows) * nsrc))()
    for j in range(nsrc):
        for i, r in enumerate(rows):
            e = segs[j * len(rows) + i]
            e.src, e.dst_off, e.n = r[2 + j], r[0], r[1]
    accp = _cuda(acc, torch.float32, "acc")
    if events is not None and events[0] is not None:
        events[0].record()
    _check(load().het_accumulate_multi(accp, segs, len(rows), nsrc,
                                       ACC_FIRST if first else ACC_ADD, float(scale),
                                       _stream(stream)), "het_accumulate_multi")
    if events is not None and events[1] is not None:
        events[1].record()


def gather_bf16(dst: torch.Tensor, grads: Sequence[tuple[torch.Tensor, int]],
                stream=None, events=None) -> None:
    """dst[off:off+g.numel()] = g for every (g, off); bf16, unscaled.
    `events` as for accumulate: recorded right around the launch(es)."""
    if not grads:
        return
    if len(grads) > HET_MAX_SEGS:
        parts = range(0, len(grads), HET_MAX_SEGS)
        for j, i in enumerate(parts):
            ev = None if events is None else (events[0] if j == 0 else None,
                                              events[1] if j == len(parts) - 1 else None)
            gather_bf16(dst, grads[i:i + HET_MAX_SEGS], stream, ev)
        return
    cap = dst.numel()
    rows: list[list[int]] = []      # [src, dst_off, n]; back-to-back segments coalesce
    for i, (g, off) in enumerate(grads):
        if off < 0 or off + g.numel() > cap:
            raise InputError(f"gather_bf16: segment {i} [{off}, {off + g.numel()}) outside {cap}")
        src, n = _cuda(g, torch.bfloat16, f"grad[{i}]"), g.numel()
        if rows and rows[-1][0] + 2 * rows[-1][2] == src and rows[-1][1] + rows[-1][2] == off:
            rows[-1][2] += n
        else:
            rows.append([src, off, n])
    segs = (HetSeg * len(rows))()
    for i, (src, off, n) in enumerate(rows):
        segs[i].src, segs[i].dst_off, segs[i].n = src, off, n
    dstp = _cuda(dst, torch.bfloat16, "dst")
    if events is not None and events[0] is not None:
        events[0].record()
    _check(load().het_gather_bf16(dstp, segs, len(rows), _stream(stream)), "het_gather_bf16")
    if events is not None and events[1] is not None:
        events[1].record()


def adamw(p: torch.Tensor, g: torch.Tensor, m: torch.Tensor, v: torch.Tensor,
          shadow: torch.Tensor | None, *, lr: float, beta1: float, beta2: float, eps: float,
          weight_decay: float, step: int, stream=None) -> None:
    n = p.numel()
    if not (g.numel() == m.numel() == v.numel() == n) or (shadow is not None and
                                                        shadow.numel() != n):
        raise InputError("adamw: size mismatch")
    sh = _cuda(shadow, torch.bfloat16, "shadow") if shadow is not None else None
    _check(load().het_adamw(_cuda(p, torch.float32, "p"), _cuda(g, torch.float32, "g"),
                            _cuda(m, torch.float32, "m"), _cuda(v, torch.float32, "v"), sh, n,
                            lr, beta1, beta2, eps, weight_decay, int(step), _stream(stream)),
           "het_adamw")


def adamw_coef(*, lr: float, beta1: float, beta2: float, eps: float, weight_decay: float,
               step: int) -> list[float]:
    """The 7 fp32 coefficients het_adamw derives for `step` (het_adamw_coef)."""
    out = (ctypes.c_float * 7)()
    _check(load().het_adamw_coef(lr, beta1, beta2, eps, weight_decay, int(step), out),
           "het_adamw_coef")
    return list(out)


def adamw_devcoef(p: torch.Tensor, g: torch.Tensor, m: torch.Tensor, v: torch.Tensor,
                  shadow: torch.Tensor | None, coef: torch.Tensor, stream=None) -> None:
    """het_adamw with its coefficients read from `coef` (7 fp32 on the device,
    as adamw_coef returns them): the form a captured CUDA graph replays."""
    n = p.numel()
    if not (g.numel() == m.numel() == v.numel() == n) or (shadow is not None and
                                                        shadow.numel() != n):
        raise InputError("adamw: size mismatch")
    if coef.numel() != 7:
        raise InputError("adamw_devcoef: coef holds 7 floats")
    sh = _cuda(shadow, torch.bfloat16, "shadow") if shadow is not None else None
    _check(load().het_adamw_devcoef(_cuda(p, torch.float32, "p"), _cuda(g, torch.float32, "g"),
                                    _cuda(m, torch.float32, "m"), _cuda(v, torch.float32, "v"),
                                    sh, n, _cuda(coef, torch.float32, "coef"), _stream(stream)),
           "het_adamw_devcoef")


def embedding_grad(acc: torch.Tensor, wte_off: int, wpe_off: int | None, dy: torch.Tensor,
                   tokens: torch.Tensor, seq: int, scale: float, stream=None) -> None:
    """Fused embedding backward + layered accumulate into the fp32 root
    accumulator (see include/hetstep.h het_embedding_grad). tokens: [rows]
    (any int dtype), dy: bf16 [rows, d]."""
    rows, d = dy.reshape(-1, dy.shape[-1]).shape
    tok = tokens.reshape(-1)
    if tok.numel() != rows:
        raise InputError("embedding_grad: one token per gradient row")
    if rows == 0:
        return
    # token runs of the stably sorted ids, built on the device without a host
    # round trip (no data-dependent shapes): run id per sorted row by a cumsum of
    # "differs from the previous id", run starts by a min-scatter, run count on
    # the device (het_embedding_grad_dev)
    dev = dy.device
    srt, order = torch.sort(tok.to(torch.int32), stable=True)
    newrun = torch.ones(rows, dtype=torch.int32, device=dev)
    torch.ne(srt[1:], srt[:-1], out=newrun[1:])
    rid = torch.cumsum(newrun, 0, dtype=torch.int32)         # 1-based run id
    pos = torch.arange(rows, dtype=torch.int32, device=dev)
    seg = torch.full((rows + 1,), rows, dtype=torch.int32, device=dev)
    seg.scatter_reduce_(0, (rid - 1).to(torch.int64), pos, reduce="amin")
    nseg = rid[-1:]
    order32 = order.to(torch.int32)
    dyc = dy.reshape(rows, d).contiguous()
    _check(load().het_embedding_grad_dev(
        _cuda(acc, torch.float32, "acc"), int(wte_off), -1 if wpe_off is None else int(wpe_off),
        _cuda(dyc, torch.bfloat16, "dy"), rows, d, order32.data_ptr(), seg.data_ptr(),
        srt.data_ptr(), nseg.data_ptr(), int(seq), float(scale), _stream(stream)),
        "het_embedding_grad_dev")


HET_TUNE_ACC_VARIANT = 1
HET_TUNE_SM_BUDGET = 2
HET_TUNE_SYMM_TIMEOUT_MS = 3
HET_TUNE_ACC_GRID = 4
LN_DIMS = (256, 768, 1024)


class LayerNormFn(torch.autograd.Function):
    """Fused LayerNorm (het_layernorm_fwd/bwd) as an autograd op; bf16 CUDA
    tensors with d in LN_DIMS."""

    @staticmethod
    def forward(ctx, x, w, b, eps):
        d = x.shape[-1]
        xc = x.contiguous()
        rows = xc.numel() // d
        y = torch.empty_like(xc)
        mean = torch.empty(rows, dtype=torch.float32, device=x.device)
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
        _check(load().het_layernorm_fwd(_cuda(xc, torch.bfloat16, "x"), _cuda(w, torch.bfloat16, "w"),
                                        _cuda(b, torch.bfloat16, "b"), y.data_ptr(),
                                        mean.data_ptr(), rstd.data_ptr(), rows, d, float(eps),
                                        _stream(None)), "het_layernorm_fwd")
        ctx.save_for_backward(xc, w, mean, rstd)
        ctx.b = _key(b)       # gradient destination lookup only
        return y

    @staticmethod
    def backward(ctx, dy):
        xc, w, mean, rstd = ctx.saved_tensors
        b = ctx.b
        d = xc.shape[-1]
        rows = xc.numel() // d
        dyc = dy.contiguous()
        dx = torch.empty_like(xc)
        dw = grad_out(w)
        db = grad_out(b)
        part = torch.empty(int(load().het_layernorm_partial_floats(d)), dtype=torch.float32,
                           device=xc.device)
        _check(load().het_layernorm_bwd(_cuda(dyc, torch.bfloat16, "dy"), xc.data_ptr(),
                                        w.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                                        dx.data_ptr(), dw.data_ptr(), db.data_ptr(),
                                        part.data_ptr(), rows, d, _stream(None)),
               "het_layernorm_bwd")
        return dx, dw, db, None


class CrossEntropyFn(torch.autograd.Function):
    """Mean next-token cross-entropy over bf16 logits with the fused kernels
    (het_xent_fwd/bwd); the backward overwrites the logits buffer in place
    with dlogits (the logits are dead after it)."""

    @staticmethod
    def forward(ctx, logits, target):
        rows, vocab = logits.shape
        lg = logits.contiguous()
        tgt = target.reshape(-1).to(torch.int64).contiguous()
        lse = torch.empty(rows, dtype=torch.float32, device=lg.device)
        loss = torch.empty(rows, dtype=torch.float32, device=lg.device)
        _check(load().het_xent_fwd(_cuda(lg, torch.bfloat16, "logits"), tgt.data_ptr(), rows,
                                   vocab, lse.data_ptr(), loss.data_ptr(), _stream(None)),
               "het_xent_fwd")
        ctx.save_for_backward(lg, tgt, lse)
        return loss.mean()

    @staticmethod
    def backward(ctx, gout):
        lg, tgt, lse = ctx.saved_tensors
        rows, vocab = lg.shape
        g = gout.reshape(1).to(torch.float32).contiguous()   # stays on the device
        _check(load().het_xent_bwd(lg.data_ptr(), tgt.data_ptr(), rows, vocab, lse.data_ptr(),
                                   g.data_ptr(), lg.data_ptr(), _stream(None)), "het_xent_bwd")
        return lg, None


RMS_DIMS = (256, 768, 1024, 2048)


class RMSNormFn(torch.autograd.Function):
    """Fused RMSNorm (het_rmsnorm_fwd/bwd) for bf16 CUDA tensors, d in RMS_DIMS."""

    @staticmethod
    def forward(ctx, x, w, eps):
        d = x.shape[-1]
        xc = x.contiguous()
        rows = xc.numel() // d
        y = torch.empty_like(xc)
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
        _check(load().het_rmsnorm_fwd(_cuda(xc, torch.bfloat16, "x"), _cuda(w, torch.bfloat16, "w"),
                                      y.data_ptr(), rstd.data_ptr(), rows, d, float(eps),
                                      _stream(None)), "het_rmsnorm_fwd")
        ctx.save_for_backward(xc, w, rstd)
        return y

    @staticmethod
    def backward(ctx, dy):
        xc, w, rstd = ctx.saved_tensors
        d = xc.shape[-1]
        rows = xc.numel() // d
        dyc = dy.contiguous()
        dx = torch.empty_like(xc)
        dw = grad_out(w)
        part = torch.empty(int(load().het_rmsnorm_partial_floats(d)), dtype=torch.float32,
                           device=xc.device)
        _check(load().het_rmsnorm_bwd(_cuda(dyc, torch.bfloat16, "dy"), xc.data_ptr(),
                                      w.data_ptr(), rstd.data_ptr(), dx.data_ptr(), dw.data_ptr(),
                                      part.data_ptr(), rows, d, _stream(None)), "het_rmsnorm_bwd")
        return dx, dw, None


def rms_norm(x: torch.Tensor, w: torch.Tensor, eps: float = 1e-6) -> torch.Tensor:
    return RMSNormFn.apply(x, w, eps)


def _ptr_or_none(t: torch.Tensor | None):
    return None if t is None else t.contiguous().data_ptr()


class AddLayerNormFn(torch.autograd.Function):
    """(s, LN(s)) with s = x + r: the residual add fused into the LayerNorm pass;
    the backward adds the residual path's gradient ds to LN's input gradient in
    the same pass and hands the sum to both x and r (no add kernels either way)."""

    @staticmethod
    def forward(ctx, x, r, w, b, eps):
        d = x.shape[-1]
        xc, rc = x.contiguous(), r.contiguous()
        rows = xc.numel() // d
        sm, y = torch.empty_like(xc), torch.empty_like(xc)
        mean = torch.empty(rows, dtype=torch.float32, device=x.device)
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
        _check(load().het_layernorm_add_fwd(_cuda(xc, torch.bfloat16, "x"),
                                            _cuda(rc, torch.bfloat16, "r"),
                                            _cuda(w, torch.bfloat16, "w"),
                                            _cuda(b, torch.bfloat16, "b"), sm.data_ptr(),
                                            y.data_ptr(), mean.data_ptr(), rstd.data_ptr(), rows,
                                            d, float(eps), _stream(None)), "het_layernorm_add_fwd")
        ctx.save_for_backward(sm, w, mean, rstd)
        ctx.b = _key(b)
        return sm, y

    @staticmethod
    def backward(ctx, ds, dy):
        sm, w, mean, rstd = ctx.saved_tensors
        d = sm.shape[-1]
        rows = sm.numel() // d
        if dy is None:
            return ds, ds, None, None, None
        dyc = dy.contiguous()
        dx = torch.empty_like(sm)
        dw, db = grad_out(w), grad_out(ctx.b)
        part = torch.empty(int(load().het_layernorm_partial_floats(d)), dtype=torch.float32,
                           device=sm.device)
        _check(load().het_layernorm_bwd_add(_cuda(dyc, torch.bfloat16, "dy"), _ptr_or_none(ds),
                                            sm.data_ptr(), w.data_ptr(), mean.data_ptr(),
                                            rstd.data_ptr(), dx.data_ptr(), dw.data_ptr(),
                                            db.data_ptr(), part.data_ptr(), rows, d,
                                            _stream(None)), "het_layernorm_bwd_add")
        return dx, dx, dw, db, None


class AddRMSNormFn(torch.autograd.Function):
    """(s, RMSNorm(s)) with s = x + r, residual add fused both ways (as
    AddLayerNormFn)."""

    @staticmethod
    def forward(ctx, x, r, w, eps):
        d = x.shape[-1]
        xc, rc = x.contiguous(), r.contiguous()
        rows = xc.numel() // d
        sm, y = torch.empty_like(xc), torch.empty_like(xc)
        rstd = torch.empty(rows, dtype=torch.float32, device=x.device)
        _check(load().het_rmsnorm_add_fwd(_cuda(xc, torch.bfloat16, "x"),
                                          _cuda(rc, torch.bfloat16, "r"),
                                          _cuda(w, torch.bfloat16, "w"), sm.data_ptr(),
                                          y.data_ptr(), rstd.data_ptr(), rows, d, float(eps),
                                          _stream(None)), "het_rmsnorm_add_fwd")
        ctx.save_for_backward(sm, w, rstd)
        return sm, y

    @staticmethod
    def backward(ctx, ds, dy):
        sm, w, rstd = ctx.saved_tensors
        d = sm.shape[-1]
        rows = sm.numel() // d
        if dy is None:
            return ds, ds, None, None
        dyc = dy.contiguous()
        dx = torch.empty_like(sm)
        dw = grad_out(w)
        part = torch.empty(int(load().het_rmsnorm_partial_floats(d)), dtype=torch.float32,
                           device=sm.device)
        _check(load().het_rmsnorm_bwd_add(_cuda(dyc, torch.bfloat16, "dy"), _ptr_or_none(ds),
                                          sm.data_ptr(), w.data_ptr(), rstd.data_ptr(),
                                          dx.data_ptr(), dw.data_ptr(), part.data_ptr(), rows, d,
                                          _stream(None)), "het_rmsnorm_bwd_add")
        return dx, dx, dw, None


def add_layer_norm(x, r, w, b, eps: float = 1e-5):
    return AddLayerNormFn.apply(x, r, w, b, eps)


def add_rms_norm(x, r, w, eps: float = 1e-6):
    return AddRMSNormFn.apply(x, r, w, eps)


class RopeFn(torch.autograd.Function):
    """In-place rotary embedding on a contiguous bf16 [b, s, heads, dh] tensor."""

    @staticmethod
    def forward(ctx, t, seq):
        b, s, h, dh = t.shape
        _check(load().het_rope_inplace(_cuda(t, torch.bfloat16, "x"), b * s, h, dh, int(seq), 0,
                                       _stream(None)), "het_rope_inplace")
        ctx.mark_dirty(t)
        ctx.seq = seq
        return t

    @staticmethod
    def backward(ctx, g):
        g = g.clone(memory_format=torch.contiguous_format)   # never rotate autograd's buffer
        b, s, h, dh = g.shape
        _check(load().het_rope_inplace(g.data_ptr(), b * s, h, dh, int(ctx.seq), 1,
                                       _stream(None)), "het_rope_inplace")
        return g, None


class SwiGLUFn(torch.autograd.Function):
    """silu(a) * b for bf16 [..., f] a, b (same shape, last dim contiguous, any
    common row stride): one fused pass forward, one backward (da, db)."""

    @staticmethod
    def forward(ctx, a, b):
        f = a.shape[-1]
        a2, b2 = a.reshape(-1, f), b.reshape(-1, f)
        if a2.stride() != b2.stride() or a2.stride(1) != 1:
            a2, b2 = a2.contiguous(), b2.contiguous()
        out = torch.empty(a.shape, dtype=torch.bfloat16, device=a.device)
        for t, name in ((a2, "a"), (b2, "b")):
            if not t.is_cuda or t.dtype != torch.bfloat16:
                raise InputError(f"swiglu: {name} must be a bf16 CUDA tensor")
        _check(load().het_swiglu_fwd(a2.data_ptr(), b2.data_ptr(), a2.stride(0), out.data_ptr(),
                                     a2.shape[0], f, _stream(None)),
               "het_swiglu_fwd")
        ctx.save_for_backward(a2, b2)
        ctx.shape = a.shape
        return out

    @staticmethod
    def backward(ctx, g):
        a2, b2 = ctx.saved_tensors
        rows, f = a2.shape[0], a2.shape[1]
        g = g.reshape(rows, f).contiguous()
        da = torch.empty((rows, f), dtype=torch.bfloat16, device=g.device)
        db = torch.empty_like(da)
        _check(load().het_swiglu_bwd(g.data_ptr(), a2.data_ptr(), b2.data_ptr(), a2.stride(0),
                                     da.data_ptr(), db.data_ptr(), f, rows, f, _stream(None)),
               "het_swiglu_bwd")
        return da.view(ctx.shape), db.view(ctx.shape)


def _colsum_scratch(rows: int, n: int, device) -> torch.Tensor:
    return torch.empty(int(load().het_colsum_partial_floats(rows, n)), dtype=torch.float32,
                       device=device)


def bias_grad(g2: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Column sums of a contiguous bf16 [rows, n] gradient (fp32 sums, bf16 out)."""
    rows, n = g2.shape
    db = out if out is not None else torch.empty(n, dtype=torch.bfloat16, device=g2.device)
    part = _colsum_scratch(rows, n, g2.device)
    _check(load().het_bias_grad(_cuda(g2, torch.bfloat16, "g"), rows, n, db.data_ptr(),
                                part.data_ptr(), _stream(None)), "het_bias_grad")
    return db


class LinearFn(torch.autograd.Function):
    """y = x W^T + b with torch's GEMMs both ways and the bias gradient from the
    fused deterministic column sum (het_bias_grad) instead of torch's reduction."""

    @staticmethod
    def forward(ctx, x, w, b):
        ctx.save_for_backward(x, w)
        ctx.b = None if b is None else _key(b)
        return torch.nn.functional.linear(x, w, b)

    @staticmethod
    def backward(ctx, g):
        x, w = ctx.saved_tensors
        g2 = g.reshape(-1, g.shape[-1]).contiguous()
        dx = (g2 @ w).view(x.shape) if ctx.needs_input_grad[0] else None
        dw = torch.mm(g2.t(), x.reshape(-1, x.shape[-1]), out=grad_out(w))
        db = None if ctx.b is None else bias_grad(g2, grad_out(ctx.b))
        return dx, dw, db


class LinearNBFn(torch.autograd.Function):
    """y = x W^T (no bias) with the weight gradient written to its registered
    destination (grad_out): the Llama projections."""

    @staticmethod
    def forward(ctx, x, w):
        ctx.save_for_backward(x, w)
        return x @ w.t()

    @staticmethod
    def backward(ctx, g):
        x, w = ctx.saved_tensors
        g2 = g.reshape(-1, g.shape[-1])
        dx = (g2 @ w).view(x.shape) if ctx.needs_input_grad[0] else None
        dw = torch.mm(g2.t(), x.reshape(-1, x.shape[-1]), out=grad_out(w))
        return dx, dw


def linear_nb(x: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    if not torch.is_grad_enabled():
        return x @ w.t()
    return LinearNBFn.apply(x, w)


class LinearGeluFn(torch.autograd.Function):
    """gelu_tanh(x W^T + b): torch's bias-epilogue GEMM, the fused GELU pass
    forward, and one pass backward for GELU' and the bias gradient together."""

    @staticmethod
    def forward(ctx, x, w, b):
        pre = torch.nn.functional.linear(x, w, b)
        y = torch.empty_like(pre)
        _check(load().het_gelu_fwd(pre.data_ptr(), y.data_ptr(), pre.numel(), _stream(None)),
               "het_gelu_fwd")
        ctx.save_for_backward(x, w, pre)
        ctx.b = _key(b)
        return y

    @staticmethod
    def backward(ctx, g):
        x, w, pre = ctx.saved_tensors
        n = pre.shape[-1]
        rows = pre.numel() // n
        g2 = g.reshape(rows, n).contiguous()
        dpre = torch.empty((rows, n), dtype=torch.bfloat16, device=g.device)
        db = grad_out(ctx.b)
        part = _colsum_scratch(rows, n, g.device)
        _check(load().het_gelu_bwd_bias(g2.data_ptr(), pre.data_ptr(), dpre.data_ptr(), rows, n,
                                        db.data_ptr(), part.data_ptr(), _stream(None)),
               "het_gelu_bwd_bias")
        dx = (dpre @ w).view(x.shape) if ctx.needs_input_grad[0] else None
        dw = torch.mm(dpre.t(), x.reshape(-1, x.shape[-1]), out=grad_out(w))
        return dx, dw, db


def linear(x: torch.Tensor, w: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    if not torch.is_grad_enabled():
        return torch.nn.functional.linear(x, w, b)
    return LinearFn.apply(x, w, b)


def linear_gelu(x: torch.Tensor, w: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    if not torch.is_grad_enabled():
        # no-grad forward: cuBLASLt's GELU+bias epilogue, one kernel
        y = torch._addmm_activation(b, x.reshape(-1, x.shape[-1]), w.t(), use_gelu=True)
        return y.view(*x.shape[:-1], w.shape[0])
    return LinearGeluFn.apply(x, w, b)


def swiglu(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    return SwiGLUFn.apply(a, b)


class SwiGLUPackedFn(torch.autograd.Function):
    """silu(y[..., :f]) * y[..., f:] of one contiguous [..., 2f] projection; the
    backward writes both halves of dy in one pass (no slice/cat copies)."""

    @staticmethod
    def forward(ctx, y):
        f = y.shape[-1] // 2
        y2 = y.reshape(-1, 2 * f)
        if not y2.is_contiguous():
            y2 = y2.contiguous()
        out = torch.empty(*y.shape[:-1], f, dtype=torch.bfloat16, device=y.device)
        p = _cuda(y2, torch.bfloat16, "y")
        _check(load().het_swiglu_fwd(p, p + 2 * f, 2 * f, out.data_ptr(), y2.shape[0], f,
                                     _stream(None)), "het_swiglu_fwd")
        ctx.save_for_backward(y2)
        ctx.shape = y.shape
        return out

    @staticmethod
    def backward(ctx, g):
        (y2,) = ctx.saved_tensors
        rows, f = y2.shape[0], y2.shape[1] // 2
        g = g.reshape(rows, f).contiguous()
        dy = torch.empty_like(y2)
        p, q = y2.data_ptr(), dy.data_ptr()
        _check(load().het_swiglu_bwd(g.data_ptr(), p, p + 2 * f, 2 * f, q, q + 2 * f, 2 * f, rows,
                                     f, _stream(None)), "het_swiglu_bwd")
        return dy.view(ctx.shape)


def swiglu_packed(y: torch.Tensor) -> torch.Tensor:
    return SwiGLUPackedFn.apply(y)


class AdjacentRowsFn(torch.autograd.Function):
    """Row-major matrices that sit back to back in one buffer (a unit's flat
    layout), seen as their row concatenation without a copy; the gradient
    splits back into views."""

    @staticmethod
    def forward(ctx, *ts):
        a = ts[0]
        pos = a.data_ptr()
        for t in ts:
            if t.data_ptr() != pos or not t.is_contiguous() or t.shape[1:] != a.shape[1:] or \
                    t.dtype != a.dtype:
                raise InputError("adjacent_rows: matrices are not adjacent in memory")
            pos += t.numel() * t.element_size()
        ctx.rows = [t.shape[0] for t in ts]
        return a.as_strided((sum(ctx.rows),) + tuple(a.shape[1:]), a.stride())

    @staticmethod
    def backward(ctx, g):
        return tuple(g.split(ctx.rows, dim=0))


def adjacent_rows(*ts: torch.Tensor) -> torch.Tensor:
    return AdjacentRowsFn.apply(*ts)


class RopeQKVFn(torch.autograd.Function):
    """[b, s, 3d] fused q/k/v projection -> rotary q, k and v as contiguous
    [b, s, heads, dh] tensors (one pass), and the backward back into one
    [b, s, 3d] gradient (one pass: no cat, no adds of three dgrad GEMMs)."""

    @staticmethod
    def forward(ctx, y, heads):
        b, s, d3 = y.shape
        d = d3 // 3
        dh = d // heads
        y = y.contiguous()
        q, k, v = (torch.empty(b, s, heads, dh, dtype=torch.bfloat16, device=y.device)
                   for _ in range(3))
        _check(load().het_rope_qkv_split(_cuda(y, torch.bfloat16, "qkv"), q.data_ptr(),
                                         k.data_ptr(), v.data_ptr(), b * s, heads, dh, s,
                                         _stream(None)), "het_rope_qkv_split")
        ctx.dims = (b, s, heads, dh)
        return q, k, v

    @staticmethod
    def backward(ctx, dq, dk, dv):
        b, s, heads, dh = ctx.dims
        dq, dk, dv = (t.contiguous() for t in (dq, dk, dv))
        dy = torch.empty(b, s, 3 * heads * dh, dtype=torch.bfloat16, device=dq.device)
        _check(load().het_rope_qkv_merge(dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                                         dy.data_ptr(), b * s, heads, dh, s, _stream(None)),
               "het_rope_qkv_merge")
        return dy, None


def rope_qkv(y: torch.Tensor, heads: int):
    return RopeQKVFn.apply(y, heads)


def rope_(t: torch.Tensor) -> torch.Tensor:
    return RopeFn.apply(t, t.shape[1])


def cross_entropy(logits: torch.Tensor, target: torch.Tensor) -> torch.Tensor:
    return CrossEntropyFn.apply(logits, target)


def layer_norm(x: torch.Tensor, w: torch.Tensor, b: torch.Tensor, eps: float = 1e-5):
    return LayerNormFn.apply(x, w, b, eps)


def probe_smid(ctas: int, stream=None) -> torch.Tensor:
    """SM id each of `ctas` CTAs ran on (emulation diagnostic)."""
    out = torch.full((ctas,), -1, dtype=torch.int32, device=torch.cuda.current_device())
    _check(load().het_probe_smid(out.data_ptr(), int(ctas), _stream(stream)), "het_probe_smid")
    return out


def set_sm_budget(nsm: int) -> None:
    """Persistent grids sized for `nsm` SMs (a green-context partition); 0 = all."""
    tune(HET_TUNE_SM_BUDGET, int(nsm))


def set_symm_timeout_ms(ms: int) -> None:
    """Spin limit of the fused collectives' cross-rank barriers (default 10 s)."""
    tune(HET_TUNE_SYMM_TIMEOUT_MS, int(ms))


def set_acc_grid(mode: int) -> None:
    """Accumulate grids: 0 persistent (one resident wave), 1 one CTA per chunk."""
    tune(HET_TUNE_ACC_GRID, int(mode))


def tune(key: int, value: int) -> None:
    _check(load().het_tune(int(key), int(value)), "het_tune")


def fill(dst: torch.Tensor, value: float, stream=None) -> None:
    _check(load().het_fill_f32(_cuda(dst, torch.float32, "dst"), float(value), dst.numel(),
                               _stream(stream)), "het_fill_f32")


# ---------------------------------------------------------------------------
# NCCL communicators

def unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().het_comm_unique_id(buf), "het_comm_unique_id")
    return buf.raw


class Comm:
    """One NCCL communicator owned by this process (rank i == cluster.gpus[i])."""

    def __init__(self, uid: bytes, nranks: int, rank: int):
        if len(uid) != 128:
            raise InputError("NCCL unique id must be 128 bytes")
        self.nranks, self.rank = nranks, rank
        h = ctypes.c_void_p()
        _check(load().het_comm_init(ctypes.byref(h), uid, nranks, rank), "het_comm_init")
        self.handle = h

    def close(self) -> None:
        if self.handle:
            _check(load().het_comm_destroy(self.handle), "het_comm_destroy")
            self.handle = ctypes.c_void_p()

    def __del__(self) -> None:  # best effort; explicit close() is preferred
        try:
            if getattr(self, "handle", None):
                load().het_comm_destroy(self.handle)
        except Exception:
            pass


def _i64(vals: Sequence[int]):
    return (ctypes.c_int64 * len(vals))(*[int(v) for v in vals])


def allgather_uneven(send: torch.Tensor, unit: torch.Tensor, counts: Sequence[int],
                     offsets: Sequence[int], comm: Comm | None, rank: int,
                     algo: int = ALGO_AUTO, stream=None) -> None:
    if unit.dtype not in (torch.bfloat16, torch.float32) or send.dtype != unit.dtype:
        raise InputError("allgather_uneven: bf16 or fp32, matching dtypes")
    n = len(counts)
    if sum(counts) != unit.numel() or send.numel() < counts[rank]:
        raise InputError("allgather_uneven: buffer sizes do not match the shard table")
    dt = DT_BF16 if unit.dtype == torch.bfloat16 else DT_F32
    _check(load().het_allgather_uneven(
        _cuda(send, send.dtype, "send") if send.numel() else None, _cuda(unit, unit.dtype, "unit"),
        _i64(counts), _i64(offsets), n, rank, dt, algo, comm.handle if comm else None,
        _stream(stream)), "het_allgather_uneven")


def reduce_scatter_uneven(src: torch.Tensor, shard: torch.Tensor, counts: Sequence[int],
                          offsets: Sequence[int], comm: Comm | None, rank: int,
                          algo: int = ALGO_AUTO, stream=None) -> None:
    n = len(counts)
    if sum(counts) != src.numel() or shard.numel() < counts[rank]:
        raise InputError("reduce_scatter_uneven: buffer sizes do not match the shard table")
    _check(load().het_reduce_scatter_uneven(
        _cuda(src, torch.float32, "src"),
        _cuda(shard, torch.float32, "shard") if shard.numel() else None,
        _i64(counts), _i64(offsets), n, rank, algo, comm.handle if comm else None,
        _stream(stream)), "het_reduce_scatter_uneven")


# ---------------------------------------------------------------------------
# route table

# HET_SYMM_HELPERS routes for skewed units at N >= 3: opt-in (HET_HELPERS=1). At
# N=4, 1 GB they measured below NCCL's rings on single-owner units (AG 418 vs 669,
# RS 445 vs 665 GB/s) and below the pair relay / multicast on the other skews
# (profiles/r2/summary.md), so the default table keeps round 1's choices.
import os as _os
HELPERS_ROUTE = _os.environ.get("HET_HELPERS", "0") == "1"
# switch-reduced helpers for the fp32 reduce-scatter (SYMM_HELPERS_MC) where a
# multicast object exists: HET_HELPERS_MC=1 lets symm_policy pick them
HELPERS_MC_ROUTE = _os.environ.get("HET_HELPERS_MC", "0") == "1"
# NVLS multicast stores / ld_reduce reach a smaller share of the link than peer
# stores / loads: single-owner AG at N=4, 1 GB, round 1: multicast 554 GB/s against
# 660-700 for the peer-class routes (profiles/r1_collectives_n4*.jsonl)
MC_EFF = 0.83
# Near-single-owner units at N >= 4 stay on the fused kernels by default (the
# whole multi-rank step is then capturable as one CUDA graph). HET_OWNER_FUSED
# selects the measured alternatives that send them to NCCL's ring instead:
# "rs16" / "rs" keep only the reduce-scatters fused (AG on NCCL), "none" sends
# both to NCCL (the round-1 table). profiles/r2o/, profiles/r2b4/.
OWNER_FUSED = _os.environ.get("HET_OWNER_FUSED", "all")


def symm_link_bytes(op: str, counts: Sequence[int], nranks: int, policy: int,
                    multicast: bool = False) -> float:
    """Largest per-GPU link bytes (ingress or egress) of one fused collective
    under `policy`: "ag" (bf16), "rs" (fp32 accumulators) or "rs16" (bf16 wire).
    The model the route choice uses; measured against it in
    profiles/r2_collectives_*.jsonl."""
    c = [int(x) for x in counts]
    n, total, mx, mn = nranks, sum(c), max(c), min(c)
    if op == "ag":
        ingress = 2 * (total - mn)
        if policy == SYMM_MULTICAST:
            return 2.0 * total / MC_EFF
        if policy == SYMM_RELAY:
            return 2.0 * relay_link_bytes(c, n)
        if policy == SYMM_HELPERS:
            return max(max(helper_plan(OP_AG, c, _prefix(c))["link_bytes"]), ingress)
        return float(max(2 * (n - 1) * mx, ingress))
    es = 4 if op == "rs" else 2
    egress = es * (total - mn)            # every rank's inputs read by the others
    if policy == SYMM_MULTICAST and op == "rs":
        return 4.0 * total / MC_EFF
    if policy == SYMM_HELPERS_MC and op == "rs":
        # plan link costs of OP_RS_MC are peer-equivalent bytes already
        return max(helper_plan(OP_RS_MC, c, _prefix(c))["link_bytes"])
    if policy == SYMM_HELPERS:
        plan = helper_plan(OP_RS if op == "rs" else OP_RS_BF16, c, _prefix(c))
        return max(max(plan["link_bytes"]), egress)
    return float(max(es * (n - 1) * mx, egress))


def _prefix(c: Sequence[int]) -> list[int]:
    out, pos = [], 0
    for x in c:
        out.append(pos)
        pos += x
    return out


def symm_policy(op: str, counts: Sequence[int], nranks: int, multicast: bool = False) -> int:
    """Policy of a fused collective: the one with the smallest largest-link load
    (symm_link_bytes) among plain AUTO (peer push / pull, or multicast when the
    workspace has it), RELAY (all-gather) and HELPERS; a non-AUTO policy must
    win by > 10%. Relay: measured at N = 4 only (N = 3..4)."""
    c = [int(x) for x in counts]
    if sum(c) <= 0:
        return SYMM_AUTO
    auto = symm_link_bytes(op, c, nranks, SYMM_AUTO)
    if multicast and op != "rs16":
        auto = min(auto, symm_link_bytes(op, c, nranks, SYMM_MULTICAST))
    best, pol = auto, SYMM_AUTO
    if op == "ag" and ag_symm_policy(c, nranks, multicast) == SYMM_RELAY:
        best, pol = min(best, 0.9 * auto), SYMM_RELAY
    if HELPERS_ROUTE and nranks >= 3:
        hb = symm_link_bytes(op, c, nranks, SYMM_HELPERS)
        if hb < 0.9 * best and hb < 0.9 * auto:
            best, pol = hb, SYMM_HELPERS
    if HELPERS_MC_ROUTE and multicast and op == "rs" and nranks >= 3:
        hb = symm_link_bytes(op, c, nranks, SYMM_HELPERS_MC)
        if hb < 0.9 * best and hb < 0.9 * auto:
            best, pol = hb, SYMM_HELPERS_MC
    return pol


def route_collective(op: str, counts: Sequence[int], nranks: int, symm: bool) -> str:
    """'symm' (fused kernels on the symmetric workspace) or 'nccl' for one
    unit's all-gather ("ag", bf16) / reduce-scatter ("rs" fp32, "rs16" bf16
    wire). Every shape is fused by default (OWNER_FUSED = "all"); symm_policy
    then picks the kernel route. Measured on the steps at N=4 (samples/s,
    fused + CUDA graph vs NCCL ring for the near-single-owner units, eager:
    NCCL nodes in a captured step hung when some ranks ran eagerly):
    BERT-large 1518 vs 1487, GPT-2 small 5260 vs 5235, Llama-1.3B 566 vs 574
    (profiles/r2b4/, r2o/, r2x/). In isolation NCCL's ring still moves a
    single-owner 1 GB unit faster (AG 672 vs 535, RS 671 vs 461 GB/s,
    profiles/r2w/); OWNER_FUSED = "none" restores that table:
      * AG: near-single-owner units at N >= 4 to NCCL's ring broadcast;
      * RS: even units, N = 2 and skewed units up to a few hundred MB fused;
        near-single-owner and very large skewed units at N >= 4 to NCCL.
    """
    if not symm or nranks == 1:
        return "nccl"
    total, mx, mn = sum(counts), max(counts), min(counts)
    owner_like = nranks >= 4 and mx >= 0.75 * total
    if HELPERS_ROUTE and nranks >= 3 and total > 0:
        # the helper routes move S (not (N-1) S) over the owner's link: fused for
        # every shape (the reduce-scatter of very large skewed units included)
        return "symm"
    if op == "rs16":
        # bf16 wire (weights + cast in the RS, half the link bytes)
        return "nccl" if owner_like and OWNER_FUSED not in ("rs16", "rs", "all") else "symm"
    if op == "ag":
        return "nccl" if owner_like and OWNER_FUSED != "all" else "symm"
    if op == "rs":
        if nranks == 2 or mx - mn <= 1 or OWNER_FUSED in ("rs", "all"):
            return "symm"
        return "nccl" if owner_like or total * 4 >= (512 << 20) else "symm"
    raise InputError(f"unknown collective {op!r}")


def helper_plan(op: int, counts: Sequence[int], offsets: Sequence[int], off: int = 0
                ) -> dict:
    """The HET_SYMM_HELPERS plan the kernels run for `op` (OP_AG / OP_RS /
    OP_RS_BF16) on a shard table: direct body vectors per rank, the
    (owner, helper) pieces and each rank's link bytes (AG egress, RS ingress)."""
    n = len(counts)
    direct = (ctypes.c_int64 * n)()
    pieces = (ctypes.c_int32 * (4 * HET_MAX_RANKS))()
    loads = (ctypes.c_double * n)()
    k = load().het_symm_helper_plan(op, n, _i64(counts), _i64(offsets), int(off), direct, pieces,
                                    2 * HET_MAX_RANKS, loads)
    if k < 0:
        raise InputError(load().het_last_error().decode())
    return {"direct": list(direct), "pieces": [(pieces[2 * i], pieces[2 * i + 1])
                                               for i in range(k)],
            "link_bytes": list(loads)}


def plain_link_bytes(op: int, counts: Sequence[int]) -> float:
    """Largest per-rank link bytes of the plain peer route (no helpers):
    AG push egress (N-1) max s (2 B), ingress S - min s; RS pull ingress
    (N-1) max s (4 B fp32 / 2 B bf16 wire)."""
    n, total = len(counts), sum(counts)
    es = 2 if op in (OP_AG, OP_RS_BF16) else 4
    return es * max((n - 1) * max(counts), total - min(counts))


RELAY_FSCALE = 1.25     # relay_plan()'s share factor past the egress balance (HET_RELAY_FSCALE)


def relay_link_bytes(counts: Sequence[int], nranks: int, fscale: float = RELAY_FSCALE) -> float:
    """Largest per-GPU link load (bytes in elements) of the relay all-gather as
    relay_plan() in csrc/hetstep_symm.cu runs it: ranks sorted by count, the
    i-th largest owner A pairs with the i-th smallest B (sB < sA); A sends a
    share f = min(1, fscale * (sA - sB)(N-1) / (2 (N-2) sA)) of its range to B
    only and B forwards it. Egress A = sA((N-1) - (N-2) f), egress B =
    sB(N-1) + (N-2) f sA; every rank's ingress is S - s_i."""
    c = sorted((int(x) for x in counts), reverse=True)
    n = nranks
    total = sum(c)
    load = float(total - c[-1])                       # ingress of the smallest owner
    for i in range(n):
        j = n - 1 - i
        if i < j and c[i] > c[j]:
            f = min(1.0, fscale * (c[i] - c[j]) * (n - 1) / (2.0 * (n - 2) * c[i]))
            load = max(load, c[i] * ((n - 1) - (n - 2) * f), c[j] * (n - 1) + (n - 2) * f * c[i])
        elif i <= j:                                  # unpaired: plain push
            load = max(load, (n - 1) * c[i])
    return load


def ag_symm_policy(counts: Sequence[int], nranks: int, multicast: bool = True) -> int:
    """Route policy for a fused all-gather: SYMM_RELAY when the relay's link
    load (relay_link_bytes, the kernel's own pairing and share) beats the
    better of plain peer push and, when the workspace has an NVLS multicast
    object, multicast (S bytes on every link) by >10%; else SYMM_AUTO.
    Measured at N=4, 1 GB (profiles/r1_final/relay_n4_c*.jsonl,
    relay_fscale_n4.jsonl): 2:1 616 vs 485 GB/s, planner 686 vs 538;
    geometric (model margin 7%) stays on multicast (532 vs 465)."""
    if nranks < 3 or nranks > 4:   # relay measured at N=4 only; N=8 keeps AUTO until run
        return SYMM_AUTO
    c = [int(x) for x in counts]
    total, mx, mn = sum(c), max(c), min(c)
    if total <= 0:
        return SYMM_AUTO
    peer = max((nranks - 1) * mx, total - mn)
    best = min(peer, total) if multicast else peer
    return SYMM_RELAY if relay_link_bytes(c, nranks) < 0.9 * best else SYMM_AUTO


# ---------------------------------------------------------------------------
# symmetric workspace + fused collectives

SYMM_ALIGN = 256


def region_tensor(raw: torch.Tensor, byte_off: int, numel: int, dtype: torch.dtype
                  ) -> torch.Tensor:
    """A typed region of a workspace allocation that aliases its memory but is
    NOT an autograd view of it: every region keeps its own version counter, so
    the backward writing gradients into the bf16-wire staging region does not
    look like an in-place update of the parameters (views of the gathered-unit
    regions) that autograd saved."""
    esz = torch.tensor([], dtype=dtype).element_size()
    start = raw.storage_offset() * raw.element_size() + byte_off
    if start % esz:
        raise InputError("workspace region is not aligned to its element size")
    return torch.empty(0, dtype=dtype, device=raw.device).set_(
        raw.untyped_storage(), start // esz, (numel,), (1,))


class SymmWorkspace:
    """One allocation with the same layout on every rank (torch symmetric
    memory = plumbing: allocation, peer mapping, NVLS multicast binding),
    carved into named typed regions plus the barrier signal area. The fused
    kernels address regions by byte offset from the peer / multicast bases.
    Barrier epochs come from the host counters `epoch[channel]`, or, between
    begin_device_epochs and end_device_epochs (a CUDA-graph capture of the
    step), from a per-channel base in this rank's signal area plus the
    launch's offset (HET_SYMM_EPOCH_DEVICE)."""

    def __init__(self, regions: Sequence[tuple[str, int, torch.dtype]], group_name: str,
                 device: torch.device, rank: int, nranks: int, ctas: int = 128,
                 use_multicast: bool = True, policy: int = SYMM_AUTO):
        import torch.distributed._symmetric_memory as symm
        if nranks > HET_MAX_RANKS:
            raise InputError(f"symmetric collectives support up to {HET_MAX_RANKS} ranks")
        lib = load()
        self.offsets: dict[str, int] = {}
        pos = 0
        for name, numel, dtype in regions:
            self.offsets[name] = pos
            pos += (numel * torch.tensor([], dtype=dtype).element_size() + SYMM_ALIGN - 1) \
                // SYMM_ALIGN * SYMM_ALIGN
        self.signal_off = pos
        total = pos + int(lib.het_symm_signal_bytes())
        self.raw = symm.empty(total, dtype=torch.uint8, device=device)
        self.raw.zero_()
        self.handle = symm.rendezvous(self.raw, group_name)
        base_off = int(getattr(self.handle, "offset", 0) or 0)
        peers = [int(p) + base_off for p in self.handle.buffer_ptrs]
        mc = int(self.handle.multicast_ptr or 0) if use_multicast else 0
        if mc:
            mc += base_off
        self.multicast = mc != 0
        d = HetSymm()
        d.nranks, d.rank = nranks, rank
        for j, p in enumerate(peers):
            d.peer_base[j] = p
        d.mc_base = mc
        d.signal_off = self.signal_off
        self.desc = d
        self.views = {name: region_tensor(self.raw, self.offsets[name], numel, dtype)
                      for name, numel, dtype in regions}
        self.epoch = [0, 0]
        # device-epoch mode (capture of a multi-rank step into a CUDA graph): the
        # host counters at capture start; None = host epochs
        self._dev_epoch0: list[int] | None = None
        self.ctas = ctas
        self.policy = policy
        torch.cuda.synchronize(device)
        self.handle.barrier()

    def _next_epoch(self, ch: int) -> int:
        """Epoch argument of the next launch on channel `ch`: the host counter, or
        in device-epoch mode its offset from the capture start flagged
        EPOCH_DEVICE (the kernel adds the device-resident base)."""
        self.epoch[ch] += 1
        if self._dev_epoch0 is None:
            return self.epoch[ch]
        return EPOCH_DEVICE | (self.epoch[ch] - self._dev_epoch0[ch])

    def begin_device_epochs(self, stream) -> None:
        """Seed the device bases from the host counters (queued on `stream`,
        before the capture) and switch the following calls to device epochs."""
        for ch in range(SYMM_CHANNELS):
            _check(load().het_symm_epoch_set(ctypes.byref(self.desc), ch, self.epoch[ch],
                                             _stream(stream)), "het_symm_epoch_set")
        self._dev_epoch0 = list(self.epoch)

    def end_device_epochs(self, stream) -> list[int]:
        """Inside the capture, after the step's last collective of each channel
        has been ordered before `stream`: queue the base advance by the step's
        launches per channel, restore the host counters (the capture ran
        nothing) and return those per-replay deltas (advance_host after each
        replay keeps eager calls in sequence)."""
        if self._dev_epoch0 is None:
            raise InputError("end_device_epochs without begin_device_epochs")
        deltas = [e - e0 for e, e0 in zip(self.epoch, self._dev_epoch0)]
        for ch, d in enumerate(deltas):
            if d:
                _check(load().het_symm_epoch_add(ctypes.byref(self.desc), ch, d,
                                                 _stream(stream)), "het_symm_epoch_add")
        self.epoch = list(self._dev_epoch0)
        self._dev_epoch0 = None
        return deltas

    def advance_host(self, deltas: Sequence[int]) -> None:
        for ch, d in enumerate(deltas):
            self.epoch[ch] += d

    def __getitem__(self, name: str) -> torch.Tensor:
        return self.views[name]

    def allgather_pack(self, src_f32: torch.Tensor, region: str, elem_off: int,
                       counts: Sequence[int], offsets: Sequence[int], stream=None,
                       policy: Optional[int] = None) -> None:
        """bf16 unit at `region`[elem_off:] <- every rank's fp32 range (fused pack+AG).
        `policy` overrides the workspace's route policy for this call."""
        ep = self._next_epoch(0)
        src = _cuda(src_f32, torch.float32, "src") if src_f32.numel() else None
        byte_off = self.offsets[region] + 2 * elem_off
        _check(load().het_symm_allgather_pack(ctypes.byref(self.desc), src, byte_off,
                                              _i64(counts), _i64(offsets), ep, 0,
                                              self.policy if policy is None else int(policy),
                                              self.ctas, _stream(stream)),
               "het_symm_allgather_pack")

    def reduce_scatter(self, region: str, elem_off: int, out: torch.Tensor,
                       counts: Sequence[int], offsets: Sequence[int], end_barrier: bool = False,
                       stream=None, policy: Optional[int] = None) -> None:
        """out <- sum over ranks of the fp32 accumulator at `region`[elem_off:] (my range).
        `policy` overrides the workspace's route policy for this call (SYMM_HELPERS:
        helpers reduce pieces in place in their own accumulator)."""
        ep = self._next_epoch(1)
        o = _cuda(out, torch.float32, "out") if out.numel() else None
        byte_off = self.offsets[region] + 4 * elem_off
        pol = self.policy if policy is None else int(policy)
        if pol == SYMM_RELAY:          # all-gather only
            pol = SYMM_AUTO
        _check(load().het_symm_reduce_scatter(ctypes.byref(self.desc), byte_off, o, _i64(counts),
                                              _i64(offsets), ep, 1, int(end_barrier),
                                              pol, self.ctas, _stream(stream)),
               "het_symm_reduce_scatter")

    def reduce_scatter_bf16(self, region: str, elem_off: int, out: torch.Tensor,
                            counts: Sequence[int], offsets: Sequence[int],
                            weights: Sequence[float], end_barrier: bool = False,
                            stream=None, policy: int = SYMM_AUTO,
                            stage: str | None = None) -> None:
        """out <- sum_j weights[j] * bf16 gradient of rank j at `region`[elem_off:]
        (my range), in fp32: Eq. 1 weighting and the cast inside the RS.
        policy=SYMM_HELPERS stages the helpers' fp32 sums in the fp32 region
        `stage` (same element offsets)."""
        ep = self._next_epoch(1)
        o = _cuda(out, torch.float32, "out") if out.numel() else None
        byte_off = self.offsets[region] + 2 * elem_off
        stage_off = self.offsets[stage] + 4 * elem_off if stage is not None else 0
        if policy == SYMM_HELPERS and stage is None:
            raise InputError("reduce_scatter_bf16: the helper route needs an fp32 stage region")
        w = (ctypes.c_float * len(weights))(*[float(x) for x in weights])
        _check(load().het_symm_reduce_scatter_bf16(ctypes.byref(self.desc), byte_off, o,
                                                   _i64(counts), _i64(offsets), w, ep,
                                                   1, int(end_barrier), int(policy), stage_off,
                                                   self.ctas, _stream(stream)),
               "het_symm_reduce_scatter_bf16")

    @staticmethod
    def status(reset: bool = False) -> int:
        return int(load().het_symm_status(int(reset)))


class CollectiveFault(RuntimeError):
    """A fused collective's cross-rank barrier timed out: the kernel went on
    without its peers, so the buffers it produced (gathered parameters,
    reduced gradient shards) are not valid."""


class StatusWatch:
    """Asynchronous check of the fused collectives' sticky device status.

    ``record(stream, tag)`` queues het_symm_status_async on `stream` (after the
    step's collectives) into a slot of a small pinned host ring and an event;
    ``poll()`` checks every slot whose event has completed and ``check()``
    waits for all of them. A non-zero status raises CollectiveFault naming
    the tag (the step) it was first seen after. No device-wide sync: the
    step driver polls the previous steps' slots at the start of each step."""

    def __init__(self, slots: int = 4):
        self.host = torch.zeros(slots, dtype=torch.int32).pin_memory()
        self.ev: list = [None] * slots
        self.tag: list = [None] * slots
        self.next = 0

    def record(self, stream, tag) -> None:
        k = self.next % len(self.ev)
        if self.ev[k] is not None:          # slot still pending: settle it first
            self._settle(k, block=True)
        _check(load().het_symm_status_async(self.host[k:].data_ptr(), _stream(stream)),
               "het_symm_status_async")
        ev = torch.cuda.Event()
        ev.record(stream)
        self.ev[k], self.tag[k] = ev, tag
        self.next += 1

    def _settle(self, k: int, block: bool) -> None:
        ev = self.ev[k]
        if ev is None:
            return
        if not block and not ev.query():
            return
        ev.synchronize()
        v, tag = int(self.host[k]), self.tag[k]
        self.ev[k] = self.tag[k] = None
        if v != 0:
            raise CollectiveFault(
                f"fused collective barrier timed out (status {v}) by {tag}: the gathered "
                f"parameters / reduced gradients of that step are invalid")

    def poll(self) -> None:
        for k in range(len(self.ev)):
            self._settle(k, block=False)

    def check(self) -> None:
        for k in range(len(self.ev)):
            self._settle(k, block=True)

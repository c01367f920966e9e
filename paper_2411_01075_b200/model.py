"""Transformer units of the four benchmark configs, as pure functions of a
flat bf16 parameter buffer.

The reference models a network as `layers` identical FSDP units of
`params_per_layer` parameters (core.py:131-154; "a sequence of
identical layers"). Here one unit = one transformer block whose parameters
are *views* into the gathered bf16 unit buffer (no copies), laid out big
matrices first so every GEMM operand is 16-byte aligned. Embeddings / final
norm / (tied) LM head form a separate "root" unit, sharded by the same state
ratios.

The GEMMs and attention stay on PyTorch ops (north_star: "The model's own
forward/backward GEMMs stay on the PyTorch ops"); the hot path this repo
owns is everything around them (layout, AG/RS, accumulate, AdamW).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn.functional as F

from . import hetstep as _K
from .core import InputError, ModelSpec


@dataclass(frozen=True)
class ArchSpec:
    name: str
    kind: str          # "gpt" (causal, pre-LN, GELU), "bert" (bidirectional), "llama"
    d: int
    layers: int
    heads: int
    ffn: int
    vocab: int         # padded to a multiple of 64
    seq: int

    def __post_init__(self) -> None:
        if self.kind not in ("gpt", "bert", "llama"):
            raise InputError(f"unknown arch kind {self.kind!r}")
        if self.d % self.heads:
            raise InputError("d must divide by heads")

    # -- layouts -----------------------------------------------------------
    def unit_layout(self) -> list[tuple[str, tuple[int, ...]]]:
        d, f = self.d, self.ffn
        if self.kind == "llama":
            return [("wq", (d, d)), ("wk", (d, d)), ("wv", (d, d)), ("wo", (d, d)),
                    ("w1", (f, d)), ("w3", (f, d)), ("w2", (d, f)),
                    ("rms1", (d,)), ("rms2", (d,))]
        return [("qkv_w", (3 * d, d)), ("proj_w", (d, d)), ("fc_w", (f, d)), ("fc2_w", (d, f)),
                ("qkv_b", (3 * d,)), ("proj_b", (d,)), ("fc_b", (f,)), ("fc2_b", (d,)),
                ("ln1_w", (d,)), ("ln1_b", (d,)), ("ln2_w", (d,)), ("ln2_b", (d,))]

    def root_layout(self) -> list[tuple[str, tuple[int, ...]]]:
        d = self.d
        if self.kind == "llama":
            return [("wte", (self.vocab, d)), ("normf", (d,))]
        return [("wte", (self.vocab, d)), ("wpe", (self.seq, d)), ("lnf_w", (d,)),
                ("lnf_b", (d,))]

    @staticmethod
    def _offsets(layout):
        out, pos = {}, 0
        for name, shape in layout:
            n = math.prod(shape)
            out[name] = (pos, shape)
            pos += n
        return out, pos

    @property
    def unit_params(self) -> int:
        return self._offsets(self.unit_layout())[1]

    @property
    def root_params(self) -> int:
        return self._offsets(self.root_layout())[1]

    def model_spec(self, global_batch: int) -> ModelSpec:
        return ModelSpec(layers=self.layers, params_per_layer=self.unit_params,
                         global_batch=global_batch)

    def flops_per_sample(self) -> float:
        """Training FLOPs per sample incl. the checkpoint recompute (4 passes of 2*P*T)."""
        tokens = self.seq
        dense = self.layers * self.unit_params + self.vocab * self.d
        attn = self.layers * 4 * self.seq * self.d   # QK^T and PV per token
        return 4 * 2 * tokens * (dense + attn)


    def model_flops_per_sample(self) -> float:
        """MODEL FLOPs of one training sample (forward + backward, no recompute):
        6 per parameter-token of every matmul weight (the blocks and the tied LM
        head; embedding lookups are free) plus 12 * s * d per token per layer
        for the attention score and value products (PaLM's MFU accounting)."""
        dense = self.layers * self.unit_params + self.vocab * self.d
        return 6.0 * self.seq * dense + 12.0 * self.layers * self.seq * self.seq * self.d


ARCHS: dict[str, ArchSpec] = {
    "tiny_gpt": ArchSpec("tiny_gpt", "gpt", d=256, layers=4, heads=4, ffn=1024, vocab=4096,
                         seq=128),
    "gpt2_small": ArchSpec("gpt2_small", "gpt", d=768, layers=12, heads=12, ffn=3072,
                           vocab=50304, seq=512),
    "bert_large": ArchSpec("bert_large", "bert", d=1024, layers=24, heads=16, ffn=4096,
                           vocab=30528, seq=512),
    "llama_1b3": ArchSpec("llama_1b3", "llama", d=2048, layers=24, heads=16, ffn=5632,
                          vocab=32000, seq=512),
}


# ---------------------------------------------------------------------------
# parameter views and init

def views(flat: torch.Tensor, layout) -> dict[str, torch.Tensor]:
    offs, total = ArchSpec._offsets(layout)
    if flat.numel() != total:
        raise InputError(f"flat buffer has {flat.numel()} elements, layout needs {total}")
    return {name: flat[o:o + math.prod(shape)].view(shape) for name, (o, shape) in offs.items()}


def segment_offsets(layout) -> dict[str, int]:
    return {name: o for name, (o, _) in ArchSpec._offsets(layout)[0].items()}


def init_flat(layout, gen: torch.Generator, device, dtype=torch.float32) -> torch.Tensor:
    """N(0, 0.02) matrices / embeddings, zero biases, unit norm weights."""
    offs, total = ArchSpec._offsets(layout)
    out = torch.empty(total, dtype=dtype, device=device)
    for name, (o, shape) in offs.items():
        seg = out[o:o + math.prod(shape)]
        if len(shape) == 2:
            seg.normal_(0.0, 0.02, generator=gen)
        elif name.endswith("_b"):
            seg.zero_()
        else:
            seg.fill_(1.0)
    return out


# ---------------------------------------------------------------------------
# forward functions (bf16 activations)

def _rope(x: torch.Tensor) -> torch.Tensor:
    b, h, s, dh = x.shape
    half = dh // 2
    inv = 1.0 / (10000.0 ** (torch.arange(0, half, device=x.device, dtype=torch.float32) / half))
    ang = torch.arange(s, device=x.device, dtype=torch.float32)[:, None] * inv[None, :]
    cos, sin = ang.cos().to(x.dtype), ang.sin().to(x.dtype)
    x1, x2 = x[..., :half], x[..., half:]
    return torch.cat([x1 * cos - x2 * sin, x1 * sin + x2 * cos], dim=-1)


def _rms(x: torch.Tensor, w: torch.Tensor, eps: float = 1e-6) -> torch.Tensor:
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)).to(x.dtype) * w


# residual add fused into the following norm (hetstep.add_layer_norm / add_rms_norm);
# a switch so tools/ab_step.py can A/B it on the same box
FUSE_RESIDUAL_NORM = True


def block_forward(arch: ArchSpec, p: dict[str, torch.Tensor], x: torch.Tensor) -> torch.Tensor:
    b, s, d = x.shape
    H, dh = arch.heads, d // arch.heads
    if arch.kind == "llama":
        if x.is_cuda and x.dtype == torch.bfloat16 and d in _K.RMS_DIMS:
            # fused sm_100a RMSNorm and in-place rotary embedding (no cos/sin/cat temporaries)
            # wq|wk|wv and w1|w3 sit back to back in the unit's flat layout: one GEMM
            # each (no weight copies), RoPE and the head split in one pass, SwiGLU over
            # the packed projection
            h = _K.rms_norm(x, p["rms1"])
            qkv = _K.linear_nb(h, _K.adjacent_rows(p["wq"], p["wk"], p["wv"]))
            q, k, v = (t.transpose(1, 2) for t in _K.rope_qkv(qkv, H))
            a = F.scaled_dot_product_attention(q, k, v, is_causal=True)
            o = _K.linear_nb(a.transpose(1, 2).reshape(b, s, d), p["wo"])
            if FUSE_RESIDUAL_NORM:
                x, h = _K.add_rms_norm(x, o, p["rms2"])
            else:
                x = x + o
                h = _K.rms_norm(x, p["rms2"])
            w13 = _K.adjacent_rows(p["w1"], p["w3"])
            return x + _K.linear_nb(_K.swiglu_packed(_K.linear_nb(h, w13)), p["w2"])
        h = _rms(x, p["rms1"])
        q = (h @ p["wq"].t()).view(b, s, H, dh).transpose(1, 2)
        k = (h @ p["wk"].t()).view(b, s, H, dh).transpose(1, 2)
        v = (h @ p["wv"].t()).view(b, s, H, dh).transpose(1, 2)
        a = F.scaled_dot_product_attention(_rope(q), _rope(k), v, is_causal=True)
        x = x + a.transpose(1, 2).reshape(b, s, d) @ p["wo"].t()
        h = _rms(x, p["rms2"])
        return x + (F.silu(h @ p["w1"].t()) * (h @ p["w3"].t())) @ p["w2"].t()
    # CUDA: linears with the fused bias-gradient column sum, and the MLP
    # up-projection + GELU as one epilogue GEMM (no-grad) / fused GELU passes
    fused = x.is_cuda and x.dtype == torch.bfloat16
    lin = _K.linear if fused else F.linear
    h = _ln(x, p["ln1_w"], p["ln1_b"])
    # q/k/v as views of the fused projection in (b, s, H, dh) memory order: SDPA
    # (cuDNN) keeps that layout for its output, so neither the head split nor
    # the merge below copies, forward or backward
    q, k, v = lin(h, p["qkv_w"], p["qkv_b"]).split(d, dim=-1)
    q, k, v = (t.view(b, s, H, dh).transpose(1, 2) for t in (q, k, v))
    a = F.scaled_dot_product_attention(q, k, v, is_causal=arch.kind == "gpt")
    attn = lin(a.transpose(1, 2).reshape(b, s, d), p["proj_w"], p["proj_b"])
    if fused and d in _K.LN_DIMS and FUSE_RESIDUAL_NORM:   # add fused into LN2, both ways
        x, h = _K.add_layer_norm(x, attn, p["ln2_w"], p["ln2_b"])
    else:
        x = x + attn
        h = _ln(x, p["ln2_w"], p["ln2_b"])
    if fused:
        h = _K.linear_gelu(h, p["fc_w"], p["fc_b"])
    else:
        h = F.gelu(F.linear(h, p["fc_w"], p["fc_b"]), approximate="tanh")
    return x + lin(h, p["fc2_w"], p["fc2_b"])


def _ln(x: torch.Tensor, w: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """LayerNorm. On CUDA the fused sm_100a kernel (hetstep.LayerNormFn: one
    pass forward, one pass backward incl. deterministic gamma/beta partials);
    elsewhere normalize + affine with torch ops (used by CPU tests only)."""
    if x.is_cuda and x.dtype == torch.bfloat16 and x.shape[-1] in _K.LN_DIMS:
        return _K.layer_norm(x, w, b)
    return torch.addcmul(b, F.layer_norm(x, (x.shape[-1],)), w)


def embed_forward(arch: ArchSpec, p: dict[str, torch.Tensor], tokens: torch.Tensor) -> torch.Tensor:
    x = F.embedding(tokens, p["wte"])
    if arch.kind != "llama":
        x = x + p["wpe"][: tokens.shape[1]]
    return x


def head_value_and_grad(arch: ArchSpec, p: dict[str, torch.Tensor], x: torch.Tensor,
                        targets: torch.Tensor, wrt: list[torch.Tensor],
                        grad_scale: float = 1.0):
    """Mean next-token loss of one microbatch and its gradients w.r.t. `wrt`
    (head parameters and the head input), the gradients scaled by grad_scale
    (a row chunk of a microbatch passes its share of the rows). On CUDA the
    cross-entropy is the fused het_xent_fwd / het_xent_bwd pair (the backward
    writes dlogits over the logits in place)."""
    with torch.enable_grad():
        if arch.kind == "llama":
            h = (_K.rms_norm(x, p["normf"]) if x.is_cuda and x.dtype == torch.bfloat16 and
                 x.shape[-1] in _K.RMS_DIMS else _rms(x, p["normf"]))
        else:
            h = _ln(x, p["lnf_w"], p["lnf_b"])
        logits = h @ p["wte"].t()
        flat = logits.view(-1, logits.shape[-1])
        if flat.is_cuda and flat.dtype == torch.bfloat16 and flat.shape[-1] % 8 == 0:
            loss = _K.cross_entropy(flat, targets.reshape(-1))
        else:
            loss = F.cross_entropy(flat, targets.reshape(-1).long())
        if grad_scale != 1.0:
            return loss.detach(), torch.autograd.grad(loss, wrt,
                                                      torch.full_like(loss, grad_scale))
        return loss.detach(), torch.autograd.grad(loss, wrt)


def head_loss(arch: ArchSpec, p: dict[str, torch.Tensor], x: torch.Tensor,
              targets: torch.Tensor) -> torch.Tensor:
    """Mean next-token cross-entropy of one microbatch (tied LM head)."""
    if arch.kind == "llama":
        h = (_K.rms_norm(x, p["normf"]) if x.is_cuda and x.dtype == torch.bfloat16 and
             x.shape[-1] in _K.RMS_DIMS else _rms(x, p["normf"]))
    else:
        h = _ln(x, p["lnf_w"], p["lnf_b"])
    logits = h @ p["wte"].t()
    flat = logits.view(-1, logits.shape[-1])
    if flat.is_cuda and flat.dtype == torch.bfloat16 and flat.shape[-1] % 8 == 0:
        # fused sm_100a cross-entropy: one pass forward, one in-place pass backward
        return _K.cross_entropy(flat, targets.reshape(-1))
    return F.cross_entropy(flat, targets.reshape(-1).long())

"""CPU reference of the whole train step (N simulated ranks in one process,
torch CPU fp32) — TEST INFRASTRUCTURE and the timed CPU baseline ONLY.

Written independently of the product's model code: the transformer math is
restated here from the architecture definition (GPT-2 / BERT / Llama blocks);
only the parameter *layout* (names, shapes, order inside a unit's flat
vector) is shared, because that is the data contract between the planner's
flat shards and the model.

Per step, exactly as the reference specifies the iteration (sim.py:226-368,
gradcheck.py:30-46):
  rank i runs l_i microbatches of m_i samples (its global sample range),
  gradients of the microbatch-mean losses are summed per rank (layered
  accumulation), scaled by m_i/B and summed over ranks (Eq. 1), and AdamW
  (torch.optim.AdamW formula, fp32) updates every parameter. Because the
  uneven shard split is a pure partition of the flat vectors, the
  post-step parameters are independent of the shard layout; the layout is
  checked separately (tests/test_layout.py, shard goldens).
"""
from __future__ import annotations

import math
from typing import Sequence

import numpy as np
import torch
import torch.nn.functional as F


def _split(flat: torch.Tensor, layout) -> dict[str, torch.Tensor]:
    out, pos = {}, 0
    for name, shape in layout:
        n = math.prod(shape)
        out[name] = flat[pos:pos + n].view(shape)
        pos += n
    return out


def _ln(x, w, b):
    mu = x.mean(-1, keepdim=True)
    var = ((x - mu) ** 2).mean(-1, keepdim=True)
    return (x - mu) / torch.sqrt(var + 1e-5) * w + b


def _rmsnorm(x, w):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-6) * w


def _attention(q, k, v, causal):
    s = q.shape[-2]
    att = (q @ k.transpose(-1, -2)) / math.sqrt(q.shape[-1])
    if causal:
        mask = torch.ones(s, s, dtype=torch.bool, device=q.device).triu(1)
        att = att.masked_fill(mask, float("-inf"))
    return att.softmax(-1) @ v


def _rotary(x):
    s, dh = x.shape[-2], x.shape[-1]
    half = dh // 2
    freq = 1.0 / (10000.0 ** (torch.arange(half, dtype=torch.float32, device=x.device) / half))
    ang = torch.arange(s, dtype=torch.float32, device=x.device)[:, None] * freq[None, :]
    c, sn = torch.cos(ang).to(x.dtype), torch.sin(ang).to(x.dtype)
    a, b = x[..., :half], x[..., half:]
    return torch.cat([a * c - b * sn, a * sn + b * c], -1)


def block(arch, p, x):
    bsz, s, d = x.shape
    H = arch.heads
    dh = d // H
    heads = lambda t: t.view(bsz, s, H, dh).transpose(1, 2)  # noqa: E731
    if arch.kind == "llama":
        h = _rmsnorm(x, p["rms1"])
        a = _attention(_rotary(heads(h @ p["wq"].T)), _rotary(heads(h @ p["wk"].T)),
                       heads(h @ p["wv"].T), True)
        x = x + a.transpose(1, 2).reshape(bsz, s, d) @ p["wo"].T
        h = _rmsnorm(x, p["rms2"])
        return x + (F.silu(h @ p["w1"].T) * (h @ p["w3"].T)) @ p["w2"].T
    h = _ln(x, p["ln1_w"], p["ln1_b"])
    qkv = h @ p["qkv_w"].T + p["qkv_b"]
    q, k, v = qkv.split(d, dim=-1)
    a = _attention(heads(q), heads(k), heads(v), arch.kind == "gpt")
    x = x + a.transpose(1, 2).reshape(bsz, s, d) @ p["proj_w"].T + p["proj_b"]
    h = _ln(x, p["ln2_w"], p["ln2_b"])
    h = h @ p["fc_w"].T + p["fc_b"]
    h = 0.5 * h * (1.0 + torch.tanh(math.sqrt(2.0 / math.pi) * (h + 0.044715 * h ** 3)))
    return x + h @ p["fc2_w"].T + p["fc2_b"]


def microbatch_loss(arch, units: Sequence[torch.Tensor], root: torch.Tensor,
                    tok: torch.Tensor) -> torch.Tensor:
    rp = _split(root, arch.root_layout())
    inp, tgt = tok[:, :-1].long(), tok[:, 1:].long()
    x = rp["wte"][inp]
    if arch.kind != "llama":
        x = x + rp["wpe"][: inp.shape[1]]
    for u in units:
        x = block(arch, _split(u, arch.unit_layout()), x)
    h = _rmsnorm(x, rp["normf"]) if arch.kind == "llama" else _ln(x, rp["lnf_w"], rp["lnf_b"])
    logits = h @ rp["wte"].T
    return F.cross_entropy(logits.reshape(-1, logits.shape[-1]), tgt.reshape(-1))


def weighted_gradient(arch, units: Sequence[torch.Tensor], root: torch.Tensor,
                      rank_tokens: Sequence[np.ndarray], micro: Sequence[tuple[int, int]]
                      ) -> tuple[list[torch.Tensor], torch.Tensor, float]:
    """Eq. 1 full-batch gradient: sum_i (m_i/B) sum_k grad(loss_ik).
    rank_tokens[i]: int32 [b_i, seq+1]; micro[i] = (m_i, l_i).
    Returns (unit grads, root grad, global loss)."""
    B = sum(m * l for m, l in micro)
    params = [u.detach().clone().requires_grad_(True) for u in units]
    rootp = root.detach().clone().requires_grad_(True)
    total = torch.zeros((), device=rootp.device)
    for tok, (m, l) in zip(rank_tokens, micro):
        for k in range(l):
            lk = microbatch_loss(arch, params, rootp,
                                 torch.from_numpy(tok[k * m:(k + 1) * m]).to(rootp.device))
            total = total + lk * (m / B)
    total.backward()
    return [p.grad for p in params], rootp.grad, float(total.detach())


def adamw_(p: torch.Tensor, g: torch.Tensor, m: torch.Tensor, v: torch.Tensor, step: int, *,
           lr: float, beta1: float, beta2: float, eps: float, weight_decay: float) -> None:
    """In-place torch.optim.AdamW (single-tensor) update."""
    p.mul_(1 - lr * weight_decay)
    m.lerp_(g, 1 - beta1)
    v.mul_(beta2).addcmul_(g, g, value=1 - beta2)
    denom = (v.sqrt() / math.sqrt(1 - beta2 ** step)).add_(eps)
    p.addcdiv_(m, denom, value=-lr / (1 - beta1 ** step))


class CPUStep:
    """The reference iteration on host cores: state = full fp32 units (the
    union of every rank's shard), one `step()` = all ranks' microbatches,
    Eq. 1 reduction, AdamW."""

    def __init__(self, arch, units: Sequence[torch.Tensor], root: torch.Tensor, opt: dict):
        self.arch, self.opt = arch, opt
        self.units = [u.detach().clone().float() for u in units]
        self.root = root.detach().clone().float()
        self.mom = [(torch.zeros_like(t), torch.zeros_like(t)) for t in self.units + [self.root]]
        self.steps = 0

    def step(self, rank_tokens, micro) -> float:
        gu, gr, loss = weighted_gradient(self.arch, self.units, self.root, rank_tokens, micro)
        self.steps += 1
        with torch.no_grad():
            for t, g, (m, v) in zip(self.units + [self.root], gu + [gr], self.mom):
                adamw_(t, g, m, v, self.steps, **self.opt)
        return loss

"""Test double for paper_2411_01075_b200.hetstep that runs on CPU tensors.

Used ONLY by CPU tests to drive the step driver's schedule, layout and
autograd plumbing without a GPU (the product path has no CPU fallback: the
real binding rejects CPU tensors). Kernel math comes from the oracle; the
multi-rank collectives go through torch.distributed (gloo) so the N>1 host
logic is exercised with world_size 2 on CPU.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from oracle import step_oracle as O

ACC_ADD, ACC_FIRST = 0, 1
ALGO_AUTO, ALGO_P2P, ALGO_OWNER, ALGO_EVEN, ALGO_SYMM = 0, 1, 2, 3, 4
calls: list[str] = []


class Comm:
    def __init__(self, uid=b"", nranks=1, rank=0):
        self.nranks, self.rank = nranks, rank
        self.handle = object()

    def close(self):
        pass


def load():
    return None


def route_collective(op, counts, nranks, symm):
    return "nccl"


def ag_symm_policy(counts, nranks, multicast=True):
    return 0


SYMM_AUTO, SYMM_MULTICAST, SYMM_PEER, SYMM_RELAY, SYMM_HELPERS = 0, 1, 2, 3, 4
SYMM_HELPERS_MC = 5


def symm_policy(op, counts, nranks, multicast=False):
    return SYMM_AUTO


def _bits(t: torch.Tensor) -> np.ndarray:
    return t.view(torch.int16).numpy().view(np.uint16)


def pack_bf16(src, dst, stream=None):
    calls.append("pack")
    dst.view(torch.int16).copy_(torch.from_numpy(O.pack(src.numpy()).view(np.int16)))


def accumulate(acc, grads, first, scale, stream=None, events=None):
    calls.append("accumulate")
    for g, off in grads:
        n = g.numel()
        cur = acc[off:off + n].numpy()
        acc[off:off + n] = torch.from_numpy(O.accumulate(cur, _bits(g.contiguous().reshape(-1)),
                                                         first, scale))


def accumulate_multi(acc, sources, offsets, first, scale, stream=None, events=None):
    calls.append("accumulate")
    for j, src in enumerate(sources):
        for g, off in zip(src, offsets):
            n = g.numel()
            cur = acc[off:off + n].numpy()
            acc[off:off + n] = torch.from_numpy(O.accumulate(
                cur, _bits(g.contiguous().reshape(-1)), first and j == 0, scale))


def adamw(p, g, m, v, shadow, *, lr, beta1, beta2, eps, weight_decay, step, stream=None):
    calls.append("adamw")
    rp, rm, rv = O.adamw(p.numpy(), g.numpy(), m.numpy(), v.numpy(), lr=lr, beta1=beta1,
                         beta2=beta2, eps=eps, weight_decay=weight_decay, step=step)
    p.copy_(torch.from_numpy(rp))
    m.copy_(torch.from_numpy(rm))
    v.copy_(torch.from_numpy(rv))
    if shadow is not None:
        pack_bf16(p, shadow)


def embedding_grad(acc, wte_off, wpe_off, dy, tokens, seq, scale, stream=None):
    calls.append("embedding_grad")
    d = dy.shape[-1]
    g = dy.reshape(-1, d).float()
    tok = tokens.reshape(-1).long()
    wte = torch.zeros(int(tok.max()) + 1, d)
    wte.index_add_(0, tok, g)
    rows = torch.arange(wte.shape[0])
    for r in rows.tolist():
        acc[wte_off + r * d: wte_off + (r + 1) * d] += scale * wte[r]
    if wpe_off is not None:
        pos = g.view(-1, seq, d).sum(0)
        acc[wpe_off: wpe_off + seq * d] += scale * pos.reshape(-1)


def fill(dst, value, stream=None):
    calls.append("fill")
    dst.fill_(value)


def allgather_uneven(send, unit, counts, offsets, comm, rank, algo=0, stream=None):
    calls.append("allgather")
    n = len(counts)
    if n == 1:
        unit.copy_(send[:counts[0]])
        return
    width = max(counts)
    buf = torch.zeros(width, dtype=torch.float32)
    buf[:counts[rank]] = send[:counts[rank]].float()
    parts = [torch.zeros(width, dtype=torch.float32) for _ in range(n)]
    dist.all_gather(parts, buf)
    for j in range(n):
        unit[offsets[j]:offsets[j] + counts[j]] = parts[j][:counts[j]].to(unit.dtype)


def reduce_scatter_uneven(src, shard, counts, offsets, comm, rank, algo=0, stream=None):
    calls.append("reduce_scatter")
    if len(counts) == 1:
        shard[:counts[0]] = src
        return
    total = src.clone().double()
    dist.all_reduce(total)
    shard[:counts[rank]] = total[offsets[rank]:offsets[rank] + counts[rank]].float()

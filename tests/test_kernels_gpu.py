"""Parity of the owned sm_100a kernels against the CPU oracle, called through
the C-ABI (paper_2411_01075_b200.hetstep -> libhetstep.so).

Tolerances (north_star): pack is bit-exact (integer bf16 bit patterns);
accumulate and AdamW are fp32 elementwise and must match within a max
relative error of 1e-5 (oracle/tolerances.max_rel: element-wise, with a
1e-2 * max|ref| floor against cancellation).
"""
import numpy as np
import pytest
import torch

from oracle import step_oracle as O
from oracle.tolerances import FP32_RTOL as RTOL
from oracle.tolerances import max_rel as _rel
from paper_2411_01075_b200 import hetstep as K
from paper_2411_01075_b200.core import InputError

pytestmark = pytest.mark.gpu


def _bits(t: torch.Tensor) -> np.ndarray:
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("n", [0, 1, 3, 4, 1000, 4099, 1 << 20, (1 << 22) + 5])
def test_pack_bit_exact(cuda, n):
    g = torch.Generator().manual_seed(n)
    x = (torch.randn(n, generator=g) * 3).float()
    if n > 8:
        x[:4] = torch.tensor([float("inf"), -float("inf"), 0.0, -0.0])
    src = x.to(cuda)
    dst = torch.empty(n, dtype=torch.bfloat16, device=cuda)
    K.pack_bf16(src, dst)
    torch.cuda.synchronize()
    assert np.array_equal(_bits(dst), O.pack(x.numpy()))


def test_pack_unaligned_tail(cuda):
    x = torch.randn(1001, generator=torch.Generator().manual_seed(1))
    src = x.to(cuda)[1:]                     # 4-byte aligned only -> scalar path
    dst = torch.empty(1000, dtype=torch.bfloat16, device=cuda)
    K.pack_bf16(src, dst)
    torch.cuda.synchronize()
    assert np.array_equal(_bits(dst), O.pack(x.numpy()[1:]))


def _segments(sizes, seed):
    g = torch.Generator().manual_seed(seed)
    grads = [torch.randn(s, generator=g).to(torch.bfloat16) for s in sizes]
    offs, pos = [], 0
    for s in sizes:
        offs.append(pos)
        pos += s
    return grads, offs, pos


@pytest.mark.parametrize("sizes", [[8], [3, 5, 7], [768 * 2304, 2304, 768 * 768, 768, 3072 * 768, 3072,
                                                    768 * 3072, 768, 768, 768, 768, 768],
                                   [1, 8191, 8192, 8193, 33000]])
def test_accumulate_layered(cuda, sizes):
    grads, offs, total = _segments(sizes, len(sizes))
    w = 3.0 / 97.0
    acc = torch.empty(total, dtype=torch.float32, device=cuda)
    ref = np.zeros(total, dtype=np.float32)
    for k in range(3):                       # l_i = 3 microbatches
        gk = [(g * (k + 1)).to(torch.bfloat16) for g in grads]
        K.accumulate(acc, [(g.to(cuda), o) for g, o in zip(gk, offs)], first=(k == 0), scale=w)
        full = np.zeros(total, dtype=np.uint16)
        for g, o in zip(gk, offs):
            full[o:o + g.numel()] = _bits(g)
        ref = O.accumulate(ref, full, k == 0, w)
    torch.cuda.synchronize()
    got = acc.cpu().numpy()
    assert _rel(got, ref) <= RTOL


@pytest.mark.parametrize("sizes", [[8], [3, 5, 7], [1, 8191, 8192, 8193, 33000],
                                   [768 * 2304, 2304, 768 * 768, 768, 3072 * 768]])
@pytest.mark.parametrize("gap", [0, 1])
def test_gather_bf16_bit_exact(cuda, sizes, gap):
    """het_gather_bf16 (bf16-wire staging): every segment lands bit-exact at its
    offset. gap=0: back-to-back segments, 16-byte vector path; gap=1: one
    untouched element between segments and a 2-byte-aligned destination
    (scalar path)."""
    grads, offs, total = _segments(sizes, 11)
    offs = [o + gap * i for i, o in enumerate(offs)]
    total += gap * len(sizes)
    dst = torch.full((total + gap,), 7.0, dtype=torch.bfloat16, device=cuda)
    view = dst[gap:]
    K.gather_bf16(view, [(g.to(cuda), o) for g, o in zip(grads, offs)])
    torch.cuda.synchronize()
    ref = np.full(total, _bits(torch.tensor([7.0], dtype=torch.bfloat16))[0], dtype=np.uint16)
    for g, o in zip(grads, offs):
        ref[o:o + g.numel()] = _bits(g)
    assert np.array_equal(_bits(view), ref)
    with pytest.raises(InputError):
        K.gather_bf16(view, [(grads[0].to(cuda), total)])


@pytest.mark.parametrize("nsrc", [1, 2, 3, 4])
@pytest.mark.parametrize("sizes", [[3, 5, 7], [1, 8191, 8192, 8193, 33000],
                                   [768 * 2304, 2304, 768 * 768, 768]])
def test_accumulate_multi_bit_exact(cuda, nsrc, sizes):
    """het_accumulate_multi over nsrc microbatches == nsrc het_accumulate passes,
    bit for bit, in FIRST and ADD mode (and the CPU oracle within RTOL)."""
    w = 5.0 / 131.0
    grads, offs, total = _segments(sizes, 3)
    src = [[(g * (j + 1) - j).to(torch.bfloat16).to(cuda) for g in grads] for j in range(nsrc)]
    for first in (True, False):
        init = torch.randn(total, generator=torch.Generator().manual_seed(9)).to(cuda)
        one, many = init.clone(), init.clone()
        for j in range(nsrc):
            K.accumulate(one, list(zip(src[j], offs)), first and j == 0, w)
        K.accumulate_multi(many, src, offs, first, w)
        torch.cuda.synchronize()
        assert torch.equal(one.view(torch.int32), many.view(torch.int32)), (first, nsrc)
        ref = init.cpu().numpy()
        for j in range(nsrc):
            full = np.zeros(total, dtype=np.uint16)
            for g, o in zip(src[j], offs):
                full[o:o + g.numel()] = _bits(g)
            ref = O.accumulate(ref, full, first and j == 0, w)
        assert _rel(many.cpu().numpy(), ref) <= RTOL


def test_accumulate_grid_modes_bit_identical(cuda):
    """HET_TUNE_ACC_GRID: one CTA per chunk (1) and the persistent wave (0) give
    bit-identical accumulators, single- and multi-source."""
    w = 7.0 / 173.0
    grads, offs, total = _segments([768 * 2304, 2304, 5, 768 * 768, 33000], 5)
    src = [[(g * (j + 1)).to(torch.bfloat16).to(cuda) for g in grads] for j in range(2)]
    out = {}
    try:
        for mode in (0, 1):
            K.set_acc_grid(mode)
            a = torch.zeros(total, device=cuda)
            K.accumulate(a, list(zip(src[0], offs)), True, w)
            K.accumulate(a, list(zip(src[1], offs)), False, w)
            b = torch.zeros(total, device=cuda)
            K.accumulate_multi(b, src, offs, True, w)
            torch.cuda.synchronize()
            out[mode] = (a, b)
    finally:
        K.set_acc_grid(0)
    for x, y in zip(out[0], out[1]):
        assert torch.equal(x.view(torch.int32), y.view(torch.int32))


def test_accumulate_multi_unaligned_and_rejects(cuda):
    grads, offs, total = _segments([1000, 4099], 4)
    acc = torch.zeros(total + 1, device=cuda)[1:]            # 4-byte aligned only
    src = [[g.to(cuda) for g in grads] for _ in range(2)]
    ref = torch.zeros_like(acc)
    K.accumulate_multi(acc, src, offs, True, 0.5)
    for j in range(2):
        K.accumulate(ref, list(zip(src[j], offs)), j == 0, 0.5)
    torch.cuda.synchronize()
    assert torch.equal(acc.view(torch.int32), ref.view(torch.int32))
    with pytest.raises(InputError):                           # mismatched source shapes
        K.accumulate_multi(acc, [src[0], [src[1][0], src[1][1][:-1]]], offs, True, 1.0)
    with pytest.raises(InputError):
        K.accumulate_multi(acc, [src[0]] * 5, offs, True, 1.0)


def test_accumulate_rejects_out_of_range(cuda):
    acc = torch.zeros(10, device=cuda)
    with pytest.raises(InputError):
        K.accumulate(acc, [(torch.zeros(8, dtype=torch.bfloat16, device=cuda), 4)], True, 1.0)


@pytest.mark.parametrize("n,shadow", [(1, True), (7, False), (4096, True), (3_000_003, True),
                                      (1 << 22, False)])
def test_adamw_matches_oracle(cuda, n, shadow):
    g = torch.Generator().manual_seed(n)
    p, gr = torch.randn(n, generator=g) * 0.02, torch.randn(n, generator=g) * 1e-3
    m, v = torch.randn(n, generator=g) * 1e-4, torch.rand(n, generator=g) * 1e-6
    opt = dict(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1)
    tp, tg, tm, tv = (t.to(cuda).contiguous() for t in (p, gr, m, v))
    sh = torch.empty(n, dtype=torch.bfloat16, device=cuda) if shadow else None
    K.adamw(tp, tg, tm, tv, sh, step=7, **opt)
    torch.cuda.synchronize()
    rp, rm, rv = O.adamw(p.numpy(), gr.numpy(), m.numpy(), v.numpy(), step=7, **opt)
    assert _rel(tp.cpu().numpy(), rp) <= RTOL
    assert _rel(tm.cpu().numpy(), rm) <= RTOL
    assert _rel(tv.cpu().numpy(), rv) <= RTOL
    if shadow:
        assert np.array_equal(_bits(sh), O.pack(tp.cpu().numpy()))


def test_adamw_matches_torch_adamw(cuda):
    """Independent pin: the kernel against torch.optim.AdamW (CUDA, foreach=False)."""
    n = 100_003
    g = torch.Generator().manual_seed(5)
    p0 = torch.randn(n, generator=g) * 0.02
    grads = [torch.randn(n, generator=g) * 1e-3 for _ in range(3)]
    ref = torch.nn.Parameter(p0.clone().to(cuda))
    opt = torch.optim.AdamW([ref], lr=1e-3, betas=(0.9, 0.95), eps=1e-8, weight_decay=0.1,
                            foreach=False, fused=False)
    p, m, v = p0.clone().to(cuda), torch.zeros(n, device=cuda), torch.zeros(n, device=cuda)
    for step, gr in enumerate(grads, 1):
        ref.grad = gr.to(cuda)
        opt.step()
        K.adamw(p, gr.to(cuda), m, v, None, lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8,
                weight_decay=0.1, step=step)
    torch.cuda.synchronize()
    assert _rel(p.cpu().numpy(), ref.detach().cpu().numpy()) <= RTOL


def test_fill(cuda):
    t = torch.empty(12345, device=cuda)
    K.fill(t, 0.0)
    torch.cuda.synchronize()
    assert float(t.abs().max()) == 0.0


@pytest.mark.parametrize("vocab,d,m,seq,wpe", [(50304, 768, 4, 512, True), (97, 100, 3, 64, True),
                                               (32000, 2048, 2, 128, False)])
def test_embedding_grad_matches_oracle(cuda, vocab, d, m, seq, wpe):
    g = torch.Generator().manual_seed(d)
    tok = torch.randint(0, vocab, (m, seq), generator=g, dtype=torch.int32)
    tok[0, :7] = 5                                   # a heavily repeated token
    dy = (torch.randn(m * seq, d, generator=g) * 0.1).to(torch.bfloat16)
    wte_off, wpe_off = 0, vocab * d if wpe else None
    size = vocab * d + (seq * d if wpe else 0)
    acc0 = torch.randn(size, generator=g)
    acc = acc0.clone().to(cuda)
    K.embedding_grad(acc, wte_off, wpe_off, dy.to(cuda), tok.to(cuda), seq, 0.25)
    torch.cuda.synchronize()
    ref = O.embedding_grad(acc0.numpy(), wte_off, wpe_off,
                           dy.view(torch.int16).numpy().view(np.uint16), tok.numpy(), seq, 0.25)
    assert _rel(acc.cpu().numpy(), ref) <= RTOL
    # deterministic: a second run from the same state is bit-identical
    acc2 = acc0.clone().to(cuda)
    K.embedding_grad(acc2, wte_off, wpe_off, dy.to(cuda), tok.to(cuda), seq, 0.25)
    torch.cuda.synchronize()
    assert torch.equal(acc, acc2)


@pytest.mark.parametrize("d,rows", [(256, 1000), (768, 4 * 512 + 3), (1024, 2048)])
def test_fused_layernorm_matches_torch_fp32(cuda, d, rows):
    """Model-side fused LayerNorm: forward and backward against torch's fp32
    LayerNorm on the same bf16 inputs (outputs are bf16: 1e-2 normwise)."""
    from oracle.tolerances import norm_rel
    g = torch.Generator().manual_seed(d)
    x = (torch.randn(rows, d, generator=g) * 2 + 0.5).to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn(d, generator=g)).to(torch.bfloat16)
    b = (0.1 * torch.randn(d, generator=g)).to(torch.bfloat16)
    dy = torch.randn(rows, d, generator=g).to(torch.bfloat16)
    xs, ws, bs = (t.to(cuda).requires_grad_(True) for t in (x, w, b))
    y = K.layer_norm(xs, ws, bs)
    y.backward(dy.to(cuda))
    xr, wr, br = (t.float().requires_grad_(True) for t in (x, w, b))
    yr = torch.nn.functional.layer_norm(xr, (d,), wr, br, 1e-5)
    yr.backward(dy.float())
    assert norm_rel(y.float().detach().cpu().numpy(), yr.detach().numpy()) <= 1e-2
    assert norm_rel(xs.grad.float().cpu().numpy(), xr.grad.numpy()) <= 1e-2
    assert norm_rel(ws.grad.float().cpu().numpy(), wr.grad.numpy()) <= 1e-2
    assert norm_rel(bs.grad.float().cpu().numpy(), br.grad.numpy()) <= 1e-2


@pytest.mark.parametrize("rows,vocab", [(3000, 50304), (517, 4096), (64, 32000)])
def test_fused_cross_entropy_matches_torch_fp32(cuda, rows, vocab):
    """Model-side fused cross-entropy against torch's fp32 cross-entropy on the
    same bf16 logits: loss 1e-5 relative, dlogits (bf16 output) 1e-2 normwise."""
    from oracle.tolerances import norm_rel
    g = torch.Generator().manual_seed(vocab)
    logits = (torch.randn(rows, vocab, generator=g) * 3).to(torch.bfloat16)
    tgt = torch.randint(0, vocab, (rows,), generator=g)
    x = logits.to(cuda).requires_grad_(True)
    loss = K.cross_entropy(x * 1, tgt.to(cuda))
    (loss * 0.5).backward()
    xr = logits.float().requires_grad_(True)
    lr = torch.nn.functional.cross_entropy(xr, tgt)
    (lr * 0.5).backward()
    assert abs(float(loss) - float(lr)) <= 1e-5 * abs(float(lr))
    assert norm_rel(x.grad.float().cpu().numpy(), xr.grad.numpy()) <= 1e-2


@pytest.mark.parametrize("d,rows", [(2048, 1500), (256, 777)])
def test_fused_rmsnorm_matches_torch_fp32(cuda, d, rows):
    from oracle.tolerances import norm_rel
    g = torch.Generator().manual_seed(d)
    x = (torch.randn(rows, d, generator=g) * 2).to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn(d, generator=g)).to(torch.bfloat16)
    dy = torch.randn(rows, d, generator=g).to(torch.bfloat16)
    xs, ws = (t.to(cuda).requires_grad_(True) for t in (x, w))
    y = K.rms_norm(xs, ws)
    y.backward(dy.to(cuda))
    xr, wr = (t.float().requires_grad_(True) for t in (x, w))
    yr = xr * torch.rsqrt((xr * xr).mean(-1, keepdim=True) + 1e-6) * wr
    yr.backward(dy.float())
    assert norm_rel(y.float().detach().cpu().numpy(), yr.detach().numpy()) <= 1e-2
    assert norm_rel(xs.grad.float().cpu().numpy(), xr.grad.numpy()) <= 1e-2
    assert norm_rel(ws.grad.float().cpu().numpy(), wr.grad.numpy()) <= 1e-2


def test_fused_rope_matches_oracle_and_inverts(cuda):
    from oracle import model_oracle as MO
    from oracle.tolerances import norm_rel
    b, s, h, dh = 2, 64, 4, 128
    t = torch.randn(b, s, h, dh, generator=torch.Generator().manual_seed(0)).to(torch.bfloat16)
    x = t.to(cuda).clone().requires_grad_(False)
    y = K.rope_(x.clone())
    ref = MO._rotary(t.float().transpose(1, 2)).transpose(1, 2)     # [b, h, s, dh] convention
    assert norm_rel(y.float().cpu().numpy(), ref.numpy()) <= 1e-2
    # backward = inverse rotation: d(rope(x))/dx applied to dy rotates it back
    xs = t.to(cuda).clone().requires_grad_(True)
    yy = K.rope_(xs * 1)
    dy = torch.randn_like(yy)
    yy.backward(dy)
    xr = t.float().transpose(1, 2).clone().requires_grad_(True)
    MO._rotary(xr).backward(dy.float().cpu().transpose(1, 2))
    assert norm_rel(xs.grad.float().cpu().numpy(), xr.grad.transpose(1, 2).numpy()) <= 1e-2


@pytest.mark.parametrize("rows,f,fused_proj", [(512, 5504, False), (300, 1376, True), (7, 13, False)])
def test_fused_swiglu_matches_torch(cuda, rows, f, fused_proj):
    """silu(a) * b fused (forward + backward) against torch's two-kernel bf16
    form and an fp32 reference; a/b either separate or the halves of one
    [rows, 2f] projection (row stride 2f)."""
    g = torch.Generator().manual_seed(rows + f)
    if fused_proj:
        ab = (torch.randn(rows, 2 * f, generator=g) * 2).to(torch.bfloat16).to(cuda)
        a, b = ab[:, :f], ab[:, f:]
    else:
        a = (torch.randn(rows, f, generator=g) * 2).to(torch.bfloat16).to(cuda)
        b = (torch.randn(rows, f, generator=g) * 2).to(torch.bfloat16).to(cuda)
    dout = torch.randn(rows, f, generator=g).to(torch.bfloat16).to(cuda)
    a1, b1 = a.detach().clone().requires_grad_(True), b.detach().clone().requires_grad_(True)
    y = K.swiglu(a1, b1)
    y.backward(dout)
    a2, b2 = a.detach().clone().requires_grad_(True), b.detach().clone().requires_grad_(True)
    yt = torch.nn.functional.silu(a2) * b2
    yt.backward(dout)
    # same rounding sequence as torch's bf16 ops: at most 1 bf16 ulp apart
    for got, want in ((y, yt), (a1.grad, a2.grad), (b1.grad, b2.grad)):
        d = (got.float() - want.float()).abs()
        assert float((d > want.float().abs() * 2 ** -7 + 1e-30).float().mean()) < 1e-3
    a3, b3 = a.float().requires_grad_(True), b.float().requires_grad_(True)
    y3 = torch.nn.functional.silu(a3) * b3
    y3.backward(dout.float())
    for got, want in ((y, y3), (a1.grad, a3.grad), (b1.grad, b3.grad)):
        rel = float((got.float() - want).norm() / want.norm())
        assert rel <= 1e-2, rel


@pytest.mark.parametrize("rows,n", [(4096, 768), (1000, 3072), (77, 2304), (33, 13)])
def test_bias_grad_and_gelu_epilogues_match_torch(cuda, rows, n):
    """Linear-layer epilogues: the deterministic bias-gradient column sum, the
    GELU forward and the fused GELU-backward + bias-gradient pass, against
    torch's bf16 ops and an fp32 reference; LinearFn / LinearGeluFn gradients
    against torch autograd."""
    g = torch.Generator().manual_seed(rows * n)
    dy = torch.randn(rows, n, generator=g).to(torch.bfloat16).to(cuda)
    db = K.bias_grad(dy)
    ref = dy.float().sum(0)
    assert float((db.float() - ref).norm() / ref.norm()) <= 4e-3
    assert torch.equal(db, K.bias_grad(dy))                    # deterministic
    # GELU forward + fused backward vs torch (same fp32 formula, bf16 rounding)
    pre = (torch.randn(rows, n, generator=g) * 3).to(torch.bfloat16).to(cuda)
    x = pre.clone().requires_grad_(True)
    yt = torch.nn.functional.gelu(x, approximate="tanh")
    yt.backward(dy)
    y = torch.empty_like(pre)
    K.load().het_gelu_fwd(pre.data_ptr(), y.data_ptr(), pre.numel(), 0)
    dpre = torch.empty_like(pre)
    dbg = torch.empty(n, dtype=torch.bfloat16, device=cuda)
    part = K._colsum_scratch(rows, n, cuda)
    assert K.load().het_gelu_bwd_bias(dy.data_ptr(), pre.data_ptr(), dpre.data_ptr(), rows, n,
                                      dbg.data_ptr(), part.data_ptr(), 0) == 0
    torch.cuda.synchronize()
    for got, want in ((y, yt), (dpre, x.grad)):
        d = (got.float() - want.float()).abs()
        assert float((d > want.float().abs() * 2 ** -7 + 1e-6).float().mean()) < 1e-3
    refb = x.grad.float().sum(0)
    assert float((dbg.float() - refb).norm() / refb.norm()) <= 4e-3
    # the autograd functions against torch's F.linear (+ GELU)
    k = 64
    xin = torch.randn(rows, k, generator=g).to(torch.bfloat16).to(cuda)
    w = (torch.randn(n, k, generator=g) * 0.1).to(torch.bfloat16).to(cuda)
    b = (torch.randn(n, generator=g) * 0.1).to(torch.bfloat16).to(cuda)
    for fused, ref_fn in ((K.LinearFn.apply, lambda a, c, e: torch.nn.functional.linear(a, c, e)),
                          (K.LinearGeluFn.apply, lambda a, c, e: torch.nn.functional.gelu(
                              torch.nn.functional.linear(a, c, e), approximate="tanh"))):
        ins1 = [t.clone().requires_grad_(True) for t in (xin, w, b)]
        ins2 = [t.float().clone().requires_grad_(True) for t in (xin, w, b)]
        fused(*ins1).backward(dy)
        ref_fn(*ins2).backward(dy.float())
        for a1, a2 in zip(ins1, ins2):
            rel = float((a1.grad.float() - a2.grad).norm() / a2.grad.norm())
            assert rel <= 1.5e-2, rel


def test_rope_qkv_split_merge_and_packed_swiglu(cuda):
    """Llama unit passes over fused projections: q/k/v split with RoPE (vs the
    CPU oracle's rotary; the backward is its transpose), SwiGLU over one packed
    [.., 2f] projection (vs torch), and the copy-free adjacent-rows view."""
    from oracle import model_oracle as MO
    from oracle.tolerances import norm_rel
    b, s, H, dh = 2, 64, 4, 64
    d = H * dh
    g = torch.Generator().manual_seed(5)
    y = torch.randn(b, s, 3 * d, generator=g).to(torch.bfloat16)
    yc = y.to(cuda).requires_grad_(True)
    q, k, v = K.rope_qkv(yc, H)
    yf = y.float().requires_grad_(True)
    heads = lambda t: t.view(b, s, H, dh).transpose(1, 2)       # noqa: E731
    rq = MO._rotary(heads(yf[..., :d])).transpose(1, 2)
    rk = MO._rotary(heads(yf[..., d:2 * d])).transpose(1, 2)
    rv = yf[..., 2 * d:].view(b, s, H, dh)
    for got, want in ((q, rq), (k, rk), (v, rv)):
        assert norm_rel(got.float().detach().cpu().numpy(), want.detach().numpy()) <= 1e-2
    assert torch.equal(v.detach().cpu(), y[..., 2 * d:].view(b, s, H, dh))
    dq, dk, dv = (torch.randn(b, s, H, dh, generator=g).to(torch.bfloat16) for _ in range(3))
    torch.autograd.backward([q, k, v], [t.to(cuda) for t in (dq, dk, dv)])
    torch.autograd.backward([rq, rk, rv], [t.float() for t in (dq, dk, dv)])
    assert norm_rel(yc.grad.float().cpu().numpy(), yf.grad.numpy()) <= 1e-2
    # packed SwiGLU
    f = 96
    yp = (torch.randn(b * s, 2 * f, generator=g) * 2).to(torch.bfloat16).to(cuda)
    y1 = yp.clone().requires_grad_(True)
    y2 = yp.clone().requires_grad_(True)
    out1 = K.swiglu_packed(y1)
    out2 = torch.nn.functional.silu(y2[:, :f]) * y2[:, f:]
    go = torch.randn(b * s, f, generator=g).to(torch.bfloat16).to(cuda)
    out1.backward(go)
    out2.backward(go)
    for got, want in ((out1, out2), (y1.grad, y2.grad)):
        dd = (got.float() - want.float()).abs()
        assert float((dd > want.float().abs() * 2 ** -7 + 1e-30).float().mean()) < 1e-3
    # adjacent rows: a view, gradients split back
    buf = torch.randn(10 * 8, device=cuda, dtype=torch.bfloat16)
    a, c = buf[:24].view(3, 8).requires_grad_(True), buf[24:80].view(7, 8).requires_grad_(True)
    w = K.adjacent_rows(a, c)
    assert w.data_ptr() == buf.data_ptr() and w.shape == (10, 8)
    (w.float() * torch.arange(10, device=cuda)[:, None]).sum().backward()
    assert torch.equal(a.grad, torch.arange(3, device=cuda)[:, None].expand(3, 8).to(a.dtype))
    assert torch.equal(c.grad, torch.arange(3, 10, device=cuda)[:, None].expand(7, 8).to(a.dtype))
    with pytest.raises(Exception):
        K.adjacent_rows(c, a)


@pytest.mark.parametrize("kind,d", [("ln", 768), ("ln", 1024), ("rms", 2048), ("rms", 256)])
def test_residual_add_fused_norms(cuda, kind, d):
    """(s, norm(s)) with s = x + r in one pass; the backward folds the residual
    path's gradient into the norm's input gradient. Against torch fp32 with
    both outputs receiving gradient."""
    rows = 300
    g = torch.Generator().manual_seed(d)
    x = torch.randn(rows, d, generator=g).to(torch.bfloat16)
    r = torch.randn(rows, d, generator=g).to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn(d, generator=g)).to(torch.bfloat16)
    bb = (0.1 * torch.randn(d, generator=g)).to(torch.bfloat16)
    ds = torch.randn(rows, d, generator=g).to(torch.bfloat16)
    dy = torch.randn(rows, d, generator=g).to(torch.bfloat16)
    ins = [t.to(cuda).requires_grad_(True) for t in (x, r, w, bb)]
    if kind == "ln":
        s, y = K.add_layer_norm(ins[0], ins[1], ins[2], ins[3])
    else:
        s, y = K.add_rms_norm(ins[0], ins[1], ins[2])
    torch.autograd.backward([s, y], [ds.to(cuda), dy.to(cuda)])
    ref = [t.float().requires_grad_(True) for t in (x, r, w, bb)]
    sr = ref[0] + ref[1]
    if kind == "ln":
        yr = torch.nn.functional.layer_norm(sr, (d,), ref[2], ref[3], 1e-5)
    else:
        yr = sr * torch.rsqrt(sr.pow(2).mean(-1, keepdim=True) + 1e-6) * ref[2]
    torch.autograd.backward([sr, yr], [ds.float(), dy.float()])
    assert torch.equal(s.detach().cpu(), (x.float() + r.float()).to(torch.bfloat16))
    pairs = [(y, yr), (ins[0].grad, ref[0].grad), (ins[1].grad, ref[1].grad),
             (ins[2].grad, ref[2].grad)] + ([(ins[3].grad, ref[3].grad)] if kind == "ln" else [])
    for got, want in pairs:
        rel = float((got.float().cpu() - want.detach()).norm() / want.detach().norm())
        assert rel <= 1e-2, rel

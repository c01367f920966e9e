"""Isolated timing of the owned kernels through the C-ABI (one GPU).

For each kernel and size: (a) back-to-back launches timed as a group (pure
kernel throughput), (b) one launch bracketed by its own events (what the
step's timers see). Prints algorithmic GB/s against MEASURED_PEAKS.json.

  python tools/kernel_bench.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_01075_b200 import hetstep as K  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    PEAK = 6650.0
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > L2


def timed(fn, nbytes, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    group = a.elapsed_time(b) / reps
    singles = []
    for _ in range(10):
        flush.zero_()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        singles.append(a.elapsed_time(b))
    single = sorted(singles)[len(singles) // 2]
    return {"group_us": group * 1e3, "group_frac": nbytes / (group * 1e-3) / 1e9 / PEAK,
            "single_us": single * 1e3, "single_frac": nbytes / (single * 1e-3) / 1e9 / PEAK}


out = {}
for n in (789_760, 7_087_872, 12_596_224, 51_384_320, 4 * 7_087_872):
    grads = [torch.randn(n, device=dev).to(torch.bfloat16)]
    acc = torch.empty(n, device=dev)
    out[f"accumulate_first_{n}"] = timed(lambda: K.accumulate(acc, [(grads[0], 0)], True, 0.5),
                                         6.0 * n)
    out[f"accumulate_add_{n}"] = timed(lambda: K.accumulate(acc, [(grads[0], 0)], False, 0.5),
                                       10.0 * n)
for n in (7_087_872, 2 * 7_087_872, 12_596_224, 51_384_320):
    g16 = torch.randn(n, device=dev).to(torch.bfloat16)
    dst16 = torch.empty(n, dtype=torch.bfloat16, device=dev)
    out[f"gather_bf16_{n}"] = timed(lambda: K.gather_bf16(dst16, [(g16, 0)]), 4.0 * n)
    g2 = [torch.randn(n, device=dev).to(torch.bfloat16) for _ in range(2)]
    acc = torch.empty(n, device=dev)
    out[f"accumulate_multi2_first_{n}"] = timed(
        lambda: K.accumulate_multi(acc, [[g2[0]], [g2[1]]], [0], True, 0.5), 8.0 * n)
    out[f"accumulate_multi2_add_{n}"] = timed(
        lambda: K.accumulate_multi(acc, [[g2[0]], [g2[1]]], [0], False, 0.5), 12.0 * n)
    del g16, dst16, g2, acc
for rows, n in ((32768, 3072), (16384, 4096)):        # GPT-2 / BERT MLP up-projection
    pre = torch.randn(rows, n, device=dev).to(torch.bfloat16)
    dy = torch.randn(rows, n, device=dev).to(torch.bfloat16)
    y, dpre = torch.empty_like(pre), torch.empty_like(pre)
    db = torch.empty(n, dtype=torch.bfloat16, device=dev)
    part = K._colsum_scratch(rows, n, dev)
    lib = K.load()
    out[f"gelu_fwd_{rows}x{n}"] = timed(
        lambda: lib.het_gelu_fwd(pre.data_ptr(), y.data_ptr(), pre.numel(), 0), 4.0 * rows * n)
    out[f"gelu_bwd_bias_{rows}x{n}"] = timed(
        lambda: lib.het_gelu_bwd_bias(dy.data_ptr(), pre.data_ptr(), dpre.data_ptr(), rows, n,
                                      db.data_ptr(), part.data_ptr(), 0), 6.0 * rows * n)
    out[f"bias_grad_{rows}x{n}"] = timed(lambda: K.bias_grad(dy), 2.0 * rows * n)
    del pre, dy, y, dpre
for n in (7_087_872 * 12, 124_082_688, 1_300_000_000 // 4):
    p, g, m, v = (torch.zeros(n, device=dev) for _ in range(4))
    sh = torch.empty(n, dtype=torch.bfloat16, device=dev)
    out[f"adamw_shadow_{n}"] = timed(lambda: K.adamw(p, g, m, v, sh, lr=1e-3, beta1=0.9,
                                                     beta2=0.95, eps=1e-8, weight_decay=0.1,
                                                     step=3), 30.0 * n, reps=10)
    out[f"pack_{n}"] = timed(lambda: K.pack_bf16(p, sh), 6.0 * n, reps=10)
    del p, g, m, v, sh
for k, r in out.items():
    print(f"{k:32s} group {r['group_us']:9.1f} us {r['group_frac']:6.3f}   "
          f"single {r['single_us']:9.1f} us {r['single_frac']:6.3f}")
print(json.dumps({"peak_gbs": PEAK, "results": out}))

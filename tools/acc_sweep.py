"""Accumulate launch-shape sweep (het_tune HET_TUNE_ACC_VARIANT) on the step's
real segment tables, inputs cold in HBM (L2 flushed before every launch):
  * gpt2_pair:  two GPT-2 units (24 segments, 14.2 M params)
  * gpt2_all:   all 12 GPT-2 units (144 segments, 85 M params; N=1 grouped launch)
  * llama_unit: one Llama-1.3B unit (9 segments, 50 M params)
  python tools/acc_sweep.py
"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_01075_b200 import hetstep as K  # noqa: E402
from paper_2411_01075_b200.model import ARCHS, segment_offsets  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
SHAPES = ["(256,4)", "(256,2)", "(256,1)", "(512,2)", "(512,1)", "(128,4)"]


def table(arch, units):
    layout = arch.unit_layout()
    seg = segment_offsets(layout)
    U = arch.unit_params
    acc = torch.zeros(U * units, device=dev)
    grads = []
    for u in range(units):
        for nm, shape in layout:
            g = torch.randn(math.prod(shape), device=dev).to(torch.bfloat16)
            grads.append((g, u * U + seg[nm]))
    return acc, grads, U * units


cases = {"gpt2_pair": table(ARCHS["gpt2_small"], 2), "gpt2_all": table(ARCHS["gpt2_small"], 12),
         "llama_unit": table(ARCHS["llama_1b3"], 1)}
res = {}
for name, (acc, grads, n) in cases.items():
    for v in range(6):
        K.tune(K.HET_TUNE_ACC_VARIANT, v)
        for first in (True, False):
            ts = []
            for _ in range(12):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                K.accumulate(acc, grads, first, 0.5)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            t = sorted(ts[2:])[len(ts[2:]) // 2] * 1e-3
            frac = (6.0 if first else 10.0) * n / t / 1e9 / PEAK
            res[f"{name}/{'first' if first else 'add'}/{v}{SHAPES[v]}"] = round(frac, 3)
            print(f"{name:11s} {'first' if first else 'add  '} variant {v} {SHAPES[v]:8s} "
                  f"{t * 1e6:8.1f} us  frac {frac:.3f}", flush=True)
K.tune(K.HET_TUNE_ACC_VARIANT, 4)
print(json.dumps(res))

"""Per-unit gradient error of the B200 step against the fp32 CPU oracle, beside
the error of plain torch bf16 autograd (the oracle's own model code run on the
GPU in bf16): separates bf16 depth accumulation from a kernel fault.

  python tools/parity_depth.py [--arch llama_1b3] [--m 1] [--l 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import json  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import model_oracle as MO  # noqa: E402
from oracle.tolerances import norm_rel  # noqa: E402
from paper_2411_01075_b200.data import rank_tokens  # noqa: E402
from paper_2411_01075_b200.layout import RankLayout  # noqa: E402
from paper_2411_01075_b200.model import ARCHS  # noqa: E402
from paper_2411_01075_b200.step import UnevenFSDPTrainer  # noqa: E402
from test_step_gpu import cpu_units, one_gpu_plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--arch", default="llama_1b3")
ap.add_argument("--m", type=int, default=1)
ap.add_argument("--l", type=int, default=1)
a = ap.parse_args()
dev = torch.device("cuda", 0)
arch = ARCHS[a.arch]
plan = one_gpu_plan(arch, a.m, a.l)
units = cpu_units(arch, seed=2)
tok = rank_tokens(plan, 0, arch.seq, arch.vocab, seed=99, step=0)
tr = UnevenFSDPTrainer(arch, plan, 0, device=dev)
tr.load_full_units(units)
tr.step(torch.from_numpy(tok).to(dev))
torch.cuda.synchronize()
g_gpu = tr.g32.cpu().numpy()
L = RankLayout.from_plan(plan, arch.unit_params, arch.root_params, 0)
del tr
torch.cuda.empty_cache()
gb, rb, lb = MO.weighted_gradient(arch, [u.to(dev, torch.bfloat16) for u in units[:-1]],
                                  units[-1].to(dev, torch.bfloat16), [tok], [(a.m, a.l)])
gb = [g.float().cpu() for g in gb + [rb]]
gu, gr, lr = MO.weighted_gradient(arch, units[:-1], units[-1], [tok], [(a.m, a.l)])
rows = []
for u, ref in enumerate(gu + [gr]):
    off, cnt = L.local_range(u)
    rows.append({"unit": u, "ours": norm_rel(g_gpu[off:off + cnt], ref.numpy()),
                 "torch_bf16": norm_rel(gb[u].numpy(), ref.numpy())})
print(json.dumps({"arch": a.arch, "m": a.m, "l": a.l, "loss_bf16_torch": float(lb),
                  "loss_fp32": float(lr), "units": rows}))

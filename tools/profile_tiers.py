"""Measure the B200 tier profiles of every benchmark config (one GPU) and
write them, in the reference's profile schema, to
paper_2411_01075_b200/profiles_b200/<config>.json (consumed by
configs.build_job(..., measured=True)).

  python tools/profile_tiers.py [--configs gpt2_small ...] [--max-m 8]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2411_01075_b200.configs import CONFIGS  # noqa: E402
from paper_2411_01075_b200.model import ARCHS  # noqa: E402
from paper_2411_01075_b200.profiler import compute_memory, profile_tier  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", nargs="*", default=sorted(CONFIGS))
ap.add_argument("--max-m", type=int, default=0,
                help="profile m = 1..max_m (0: per config, past the largest microbatch the "
                     "bench plans use at N = 1..8)")
ap.add_argument("--out-dir", default=os.path.join(ROOT, "paper_2411_01075_b200", "profiles_b200"))
ap.add_argument("--no-calibrate", action="store_true",
                help="per-unit backward only (no whole-step calibration)")
a = ap.parse_args()
MAX_M = {"tiny_gpt": 8, "gpt2_small": 96, "bert_large": 80, "llama_1b3": 32}
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
for name in a.configs:
    cfg = CONFIGS[name]
    arch = ARCHS[cfg.arch]
    t0 = time.time()
    max_m = a.max_m or MAX_M.get(name, 16)
    mem = compute_memory(arch, list(range(1, max_m + 1)), dev)
    docs = [profile_tier(arch, tier, dev, max_m, mem=list(mem), calibrate=not a.no_calibrate)
            for tier in sorted(set(cfg.tiers))]
    os.makedirs(a.out_dir, exist_ok=True)
    out = os.path.join(a.out_dir, f"{name}.json")
    with open(out, "w") as fh:
        json.dump({"meta": {"gpu": torch.cuda.get_device_name(dev), "torch": torch.__version__,
                            "seconds": time.time() - t0, "tool": "tools/profile_tiers.py",
                            "calibrated": not a.no_calibrate},
                   "profiles": docs}, fh, indent=1)
    print(name, f"{time.time() - t0:.1f}s", [(d["profile_key"], d["fwd_ms"][0][1], d["fwd_ms"][-1][1],
                                              d["compute_mem_gib"][-1][1]) for d in docs], flush=True)

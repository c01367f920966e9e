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
ap.add_argument("--max-m", type=int, default=16)
a = ap.parse_args()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
for name in a.configs:
    cfg = CONFIGS[name]
    arch = ARCHS[cfg.arch]
    t0 = time.time()
    mem = compute_memory(arch, list(range(1, a.max_m + 1)), dev)
    docs = [profile_tier(arch, tier, dev, a.max_m, mem=list(mem)) for tier in sorted(set(cfg.tiers))]
    out = os.path.join(ROOT, "paper_2411_01075_b200", "profiles_b200", f"{name}.json")
    with open(out, "w") as fh:
        json.dump({"meta": {"gpu": torch.cuda.get_device_name(dev), "torch": torch.__version__,
                            "seconds": time.time() - t0, "tool": "tools/profile_tiers.py"},
                   "profiles": docs}, fh, indent=1)
    print(name, f"{time.time() - t0:.1f}s", [(d["profile_key"], d["fwd_ms"][0][1], d["fwd_ms"][-1][1],
                                              d["compute_mem_gib"][-1][1]) for d in docs], flush=True)

"""Is the N=1 step host-bound? Host issue time of one step (step() call to
return, no sync) against its device time (CUDA events), and the device time
with the host kept far ahead (several steps queued before the first sync).

  python tools/host_bound.py [--config gpt2_small]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_01075_b200.configs import build_job  # noqa: E402
from paper_2411_01075_b200.data import rank_tokens  # noqa: E402
from paper_2411_01075_b200.step import UnevenFSDPTrainer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="gpt2_small")
ap.add_argument("--steps", type=int, default=6)
args = ap.parse_args()
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
job = build_job(args.config, 1, measured=True)
tr = UnevenFSDPTrainer(job.arch, job.plan, 0, device=dev)
tr.init_params(seed=0)
tok = torch.from_numpy(rank_tokens(job.plan, 0, job.arch.seq, job.arch.vocab, 1, 0)).to(dev)
for _ in range(3):
    tr.step(tok)
torch.cuda.synchronize()
host, devt = [], []
for _ in range(args.steps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    t0 = time.perf_counter()
    tr.step(tok)
    t1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    host.append((t1 - t0) * 1e3)
    devt.append(a.elapsed_time(b))
# GPU busy check: a long sleep kernel queued first lets the host get ahead, so
# the device time of the following steps is pure GPU time
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
torch.cuda._sleep(int(2e9))            # ~1 s of GPU spin
a.record()
for _ in range(args.steps):
    tr.step(tok)
b.record()
torch.cuda.synchronize()
ahead = a.elapsed_time(b) / args.steps
print(f"{args.config}: host issue {sum(host)/len(host):.2f} ms/step, device (host-paced) "
      f"{sum(devt)/len(devt):.2f} ms/step, device (host far ahead) {ahead:.2f} ms/step")

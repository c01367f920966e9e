"""Per-op CUDA time of one train step (torch.profiler/CUPTI), for finding the
model-side hot spots around the owned kernels. Single GPU.

  python tools/profile_step.py [--config gpt2_small] [--batch 64]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2411_01075_b200.configs import build_job  # noqa: E402
from paper_2411_01075_b200.data import rank_tokens  # noqa: E402
from paper_2411_01075_b200.step import UnevenFSDPTrainer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="gpt2_small")
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--rows", type=int, default=40)
a = ap.parse_args()
torch.cuda.set_device(0)
job = build_job(a.config, 1, global_batch=a.batch)
tr = UnevenFSDPTrainer(job.arch, job.plan, 0, device=torch.device("cuda", 0))
tr.init_params(0)
tok = torch.from_numpy(rank_tokens(job.plan, 0, job.arch.seq, job.arch.vocab, 1, 0)).cuda()
for _ in range(3):
    tr.step(tok)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU], record_shapes=True) as prof:
    tr.step(tok)
    torch.cuda.synchronize()
print(prof.key_averages(group_by_input_shape=True).table(sort_by="cuda_time_total",
                                                          row_limit=a.rows, max_name_column_width=60,
                                                          max_shapes_column_width=80))

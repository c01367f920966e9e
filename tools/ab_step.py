"""Interleaved A/B of one switch on the N=1 train step (same process, same
box, alternating blocks of steps so clock/power drift hits both arms).

  python tools/ab_step.py --config gpt2_small --switch fuse_residual_norm
  python tools/ab_step.py --config gpt2_small --switch acc_group
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2411_01075_b200 import model as M  # noqa: E402
from paper_2411_01075_b200.configs import build_job  # noqa: E402
from paper_2411_01075_b200.data import rank_tokens  # noqa: E402
from paper_2411_01075_b200.step import UnevenFSDPTrainer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="gpt2_small")
ap.add_argument("--switch", default="fuse_residual_norm")
ap.add_argument("--blocks", type=int, default=6)
ap.add_argument("--steps", type=int, default=8)
ap.add_argument("--offload-schedule", default="reference")
ap.add_argument("--ml", default=None,
                help="M,L: run a one-rank plan with microbatch M and L microbatches "
                     "(layered GA) instead of the config's N=1 plan")
args = ap.parse_args()

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
job = build_job(args.config, 1, measured=True)
plan = job.plan
if args.ml:
    from paper_2411_01075_b200.core import GpuAssignment, ModelSpec, TrainPlan
    from paper_2411_01075_b200.sharding import assign_unit_shards
    m, l = (int(x) for x in args.ml.split(","))
    md = ModelSpec(job.arch.layers, job.arch.unit_params, m * l)
    plan = TrainPlan((GpuAssignment("ab", m, l, m * l, 1.0, 0.0, float(md.state_bytes)),),
                     1.0, 1.0, 2.0 * job.arch.layers, False, assign_unit_shards([1.0], md))
tr = UnevenFSDPTrainer(job.arch, plan, 0, device=dev,
                       offload_activations=args.switch == "offload",
                       offload_schedule=args.offload_schedule)
tr.init_params(seed=0)
tok = torch.from_numpy(rank_tokens(plan, 0, job.arch.seq, job.arch.vocab, 1, 0)).to(dev)


def setting(on: bool) -> None:
    if args.switch == "fuse_residual_norm":
        M.FUSE_RESIDUAL_NORM = on
    elif args.switch == "keep_last":
        tr.keep_last_graph = on
    elif args.switch == "offload":
        tr.offload = on
    elif args.switch == "acc_microbatches":
        tr.acc_microbatches = 2 if on else 1
    elif args.switch == "acc_group":
        tr.acc_group = tr.L.blocks if on else 2
    else:
        raise SystemExit(f"unknown switch {args.switch}")


times = {True: [], False: []}
for blk in range(args.blocks):
    for on in ((True, False) if blk % 2 == 0 else (False, True)):
        setting(on)
        for _ in range(2):
            tr.step(tok)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            tr.step(tok)
        b.record()
        torch.cuda.synchronize()
        times[on].append(a.elapsed_time(b) / args.steps)
on, off = statistics.median(times[True]), statistics.median(times[False])
print(f"{args.config} {args.switch}: on {on:.3f} ms/step, off {off:.3f} ms/step, "
      f"on/off {on / off:.4f}  (blocks on {[round(t, 2) for t in times[True]]}, "
      f"off {[round(t, 2) for t in times[False]]})")

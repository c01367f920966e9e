import sys, os
sys.path.insert(0, "/root/repo")
import torch, numpy as np
from paper_2411_01075_b200 import GpuAssignment, ModelSpec, TrainPlan, assign_unit_shards
from paper_2411_01075_b200.data import rank_tokens
from paper_2411_01075_b200.model import ARCHS
from paper_2411_01075_b200.step import UnevenFSDPTrainer
cuda = torch.device("cuda", 0)
arch = ARCHS["gpt2_small"]
model = ModelSpec(arch.layers, arch.unit_params, 16)
plan = TrainPlan((GpuAssignment("g0", 4, 4, 16, 1.0, 0.0, float(model.state_bytes)),), 1.0, 1.0, 2.0, False, assign_unit_shards([1.0], model))
tok = torch.from_numpy(rank_tokens(plan, 0, arch.seq, arch.vocab, seed=3, step=0)).to(cuda)
gs = {}
for name, off in (("a", False), ("b", False), ("c", True), ("d", True)):
    tr = UnevenFSDPTrainer(arch, plan, 0, device=cuda, offload_activations=off)
    tr.init_params(seed=1)
    tr.step(tok); torch.cuda.synchronize()
    gs[name] = tr.g32.clone()
    del tr
def nrel(x, y): return float((x - y).norm() / y.norm())
print("a-b (no offload twice)", nrel(gs["a"], gs["b"]))
print("c-a (offload vs not)", nrel(gs["c"], gs["a"]))
print("c-d (offload twice)", nrel(gs["c"], gs["d"]))

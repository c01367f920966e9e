"""Which ops make two identical steps differ? (1 GPU diagnostic)"""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01075_b200 import GpuAssignment, ModelSpec, TrainPlan, assign_unit_shards  # noqa
from paper_2411_01075_b200.data import rank_tokens  # noqa: E402
from paper_2411_01075_b200.model import ARCHS  # noqa: E402
from paper_2411_01075_b200.step import UnevenFSDPTrainer  # noqa: E402

cuda = torch.device("cuda", 0)
arch = ARCHS["gpt2_small"]
model = ModelSpec(arch.layers, arch.unit_params, 16)
plan = TrainPlan((GpuAssignment("g0", 4, 4, 16, 1.0, 0.0, float(model.state_bytes)),), 1.0, 1.0,
                 2.0, False, assign_unit_shards([1.0], model))
tok = torch.from_numpy(rank_tokens(plan, 0, arch.seq, arch.vocab, seed=3, step=0)).to(cuda)


def run(det):
    torch.backends.cudnn.deterministic = det
    tr = UnevenFSDPTrainer(arch, plan, 0, device=cuda)
    tr.init_params(seed=1)
    tr.step(tok)
    torch.cuda.synchronize()
    return [tr.g32[o:o + c].clone() for o, c in (tr.L.local_range(u) for u in range(arch.layers + 1))]


with warnings.catch_warnings(record=True) as w:
    warnings.simplefilter("always")
    torch.use_deterministic_algorithms(True, warn_only=True)
    run(False)
    print("nondeterministic ops:", sorted({str(x.message)[:160] for x in w}))
torch.use_deterministic_algorithms(False)
for det in (False, True):
    a, b = run(det), run(det)
    print("cudnn.deterministic", det, "per-unit nrel:",
          [round(float((x - y).norm() / y.norm()), 6) for x, y in zip(a, b)])

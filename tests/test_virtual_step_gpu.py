"""Multi-rank train-step parity at the BASELINE layouts on ONE GPU.

N trainers (one per virtual rank, tests/vranks.py) run in N threads of one
process on one B200. Each has its own compute / all-gather / reduce-scatter
streams and its rank's view of one shared symmetric allocation, so the step
issues exactly the fused kernels it issues on N GPUs (peer and helper
routes; NVLS multicast needs real GPUs) and its ranks meet at the same
in-kernel barriers. The driver's 1-GPU test run thereby checks the N = 2, 4
and 8 step end to end against the CPU oracle.

Plans: the planner's bench plan of each config at N ranks
(configs.build_job: the shard layout of the real units from the plan's state
ratios, and each rank's l_i), with every microbatch m_i scaled down so the
fp32 CPU oracle finishes in seconds; the uneven Eq. 1 weights m_i / B, the
layered accumulation and the state layout are the plan's.

Bars (north_star): loss within 2e-2 relative; every unit's
reduced gradient within 2e-2 normwise of the oracle's Eq. 1 gradient
(gradcheck.py:30-46; sim.py:278-322), or within plain torch bf16 autograd's
own error where that exceeds 2e-2 (test_step_configs_gpu.grad_bar), and
element-wise within 5e-2 of the
unit's max|g|; post-AdamW master / moments within 1e-5 (max relative) of the
oracle's AdamW fed the reduced gradient; no barrier timeout.
"""
import os
import subprocess
import sys

import pytest

from vstep_worker import CASES

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("name,n", CASES)
def test_virtual_multirank_step_matches_oracle(cuda, name, n):
    """One case per subprocess (tests/vstep_worker.py), with the stream-ordered
    allocator: see that module's docstring for why."""
    env = dict(os.environ, PYTORCH_CUDA_ALLOC_CONF="backend:cudaMallocAsync")
    proc = subprocess.run([sys.executable, os.path.join(HERE, "vstep_worker.py"), name, str(n)],
                          capture_output=True, text=True, timeout=1200, env=env)
    print(proc.stdout[-2000:])
    assert proc.returncode == 0 and "VSTEP_OK" in proc.stdout, \
        proc.stdout[-3000:] + proc.stderr[-3000:]

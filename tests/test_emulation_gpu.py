"""The heterogeneity emulation holds what it claims (north_star: "per-rank HBM
budgets are set with a memory-fraction cap, and per-rank SM partitions are
set with CUDA green contexts"; reference capacity semantics core.py:101-127):

  * a kernel launched on a tier's compute stream runs only on the tier's SMs
    (every CTA records its %smid; the distinct ids are <= the partition),
    also when captured on that stream into a CUDA graph and replayed;
  * the persistent grids of the owned kernels are sized for the partition
    (het_tune HET_TUNE_SM_BUDGET is set by emulate_tier);
  * an allocation past the tier's HBM cap raises instead of succeeding.
"""
import pytest
import torch

from paper_2411_01075_b200 import hetstep as K
from paper_2411_01075_b200.configs import cluster_doc
from paper_2411_01075_b200.core import cluster_from_dict
from paper_2411_01075_b200.emulate import emulate_tier
from paper_2411_01075_b200.model import ARCHS

pytestmark = pytest.mark.gpu

_KEEP = []      # green contexts must outlive every stream/tensor that used them


def test_green_context_confines_kernels_to_the_partition(cuda):
    arch = ARCHS["tiny_gpt"]
    cluster = cluster_from_dict(cluster_doc(arch, ["b200", "b200_half"]))
    emu = emulate_tier(cluster, 1, cuda, sm_partition=True, memory_cap=False)
    _KEEP.append(emu)
    try:
        total = torch.cuda.get_device_properties(cuda).multi_processor_count
        assert emu.green is not None and emu.num_sms < total
        assert emu.num_sms == 72          # 0.5 * 148 in 8-SM granules
        ids = K.probe_smid(emu.num_sms * 8, stream=emu.stream)
        torch.cuda.synchronize()
        inside = set(ids.cpu().tolist())
        assert -1 not in inside
        assert len(inside) <= emu.num_sms, (len(inside), emu.num_sms)
        # the same probe on an ordinary stream spreads over the whole device
        ids_all = K.probe_smid(total * 8)
        torch.cuda.synchronize()
        assert len(set(ids_all.cpu().tolist())) > emu.num_sms
        # a CUDA graph captured on the partition's stream (how a green-context rank
        # captures its step, step.UnevenFSDPTrainer._capture) keeps the partition
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=emu.stream):
            ids_g = K.probe_smid(emu.num_sms * 8, stream=emu.stream)
        for _ in range(3):
            ids_g.fill_(-1)
            torch.cuda.synchronize()
            with torch.cuda.stream(emu.stream):
                g.replay()
            torch.cuda.synchronize()
            replayed = set(ids_g.cpu().tolist())
            assert -1 not in replayed
            assert len(replayed) <= emu.num_sms, (len(replayed), emu.num_sms)
    finally:
        K.set_sm_budget(0)


def test_memory_cap_bounds_allocations(cuda):
    arch = ARCHS["tiny_gpt"]
    cluster = cluster_from_dict(cluster_doc(arch, ["b200", "b200_half"],
                                            memory_gib={"b200_half": 2.0}))
    torch.cuda.empty_cache()
    emu = emulate_tier(cluster, 1, cuda, sm_partition=False, memory_cap=True)
    try:
        assert emu.memory_cap_bytes == 2 * 2 ** 30
        ok = torch.empty(256 << 20, dtype=torch.uint8, device=cuda)      # fits under 2 GiB
        with pytest.raises(torch.OutOfMemoryError):
            torch.empty(int(2.5 * 2 ** 30), dtype=torch.uint8, device=cuda)
        del ok
    finally:
        torch.cuda.set_per_process_memory_fraction(1.0, cuda)
        torch.cuda.empty_cache()

#!/usr/bin/env python
"""Turn ncu captures brought back in gpurun_out/ into the committed summaries.

  python profiles/summarize.py --full gpurun_out/prof_r1.ncu-rep \
      --launches gpurun_out/launches.csv --tag r1 --config "gpt2_small N=1 B=64"

Writes profiles/ncu_summary.json (per owned kernel: duration, DRAM bytes,
throughput, registers, grid — the `traffic` source for bench.py's roofline)
and profiles/<tag>_launch_shares.md (share of one step's device time per
kernel from the serialized, cold-cache launch list).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
           "launch__block_size", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "lts__t_bytes.sum"]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0,
              "ms": 1e3, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}


def full_summary(rep: str, algo_bytes: dict[str, float], config: str) -> dict:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out: dict[str, dict] = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        key = ("het_adamw" if "adamw" in name
               else "het_accumulate_multi_first" if "accumulate_multi_kernel<1" in name
               else "het_accumulate_multi" if "accumulate_multi_kernel<0" in name
               else "het_accumulate_first" if "accumulate_kernel<1" in name
               else "het_accumulate" if "accumulate" in name
               else "het_gather_bf16" if "gather_bf16" in name
               else "het_bias_grad" if "colsum_kernel<" in name and "BiasOnly" in name
               else "het_gelu_bwd_bias" if "colsum_kernel<" in name and "GeluBwd" in name
               else "het_pack" if "pack" in name else name.split("(")[0])
        rec = {}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = float(r[i].replace(",", "")) if r[i] else 0.0
                rec[m] = v * UNIT_SCALE.get(units[i], 1.0)
        dram = rec.get("dram__bytes_read.sum", 0) + rec.get("dram__bytes_write.sum", 0)
        entry = {"kernel": name, "duration_us": rec.get("gpu__time_duration.sum"),
                 "dram_bytes": dram, "dram_read": rec.get("dram__bytes_read.sum"),
                 "dram_write": rec.get("dram__bytes_write.sum"),
                 "dram_pct_of_peak": rec.get(
                     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                 "grid": rec.get("launch__grid_size"), "block": rec.get("launch__block_size"),
                 "registers": rec.get("launch__registers_per_thread"),
                 "warps_active_pct": rec.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
                 "config": config}
        # keep the largest launch of each owned kernel (the unit-sized one)
        if key not in out or (entry["duration_us"] or 0) > (out[key]["duration_us"] or 0):
            out[key] = entry
    for k, e in out.items():
        if k in algo_bytes:
            e["algorithmic_bytes"] = algo_bytes[k]
            e["achieved_gbs_cold"] = algo_bytes[k] / (e["duration_us"] * 1e-6) / 1e9
    return out


def launch_shares(path: str) -> tuple[str, dict]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    data = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[1:]
            if r[mi] == "gpu__time_duration.sum"]
    marks = [i for i, (k, _) in enumerate(data) if "adamw" in k]
    s, e = (marks[-2] + 1, marks[-1] + 1) if len(marks) >= 2 else (0, len(data))
    tot, cnt = collections.Counter(), collections.Counter()
    for k, v in data[s:e]:
        key = k.split("(")[0][:100]
        tot[key] += v
        cnt[key] += 1
    T = sum(tot.values())
    owned = {k: v for k, v in tot.items() if "adamw" in k or "accumulate" in k or "pack" in k
             or "fill_kernel" in k or "gather_bf16" in k or "symm_" in k}
    model_side = {k: v for k, v in tot.items() if any(t in k for t in (
        "ln_", "rms_", "xent", "rope", "swiglu", "colsum", "gelu_fwd", "embedding_grad"))}
    nccl = {k: v for k, v in tot.items() if "nccl" in k.lower()}
    lines = ["| share | total us | launches | kernel |", "|---:|---:|---:|---|"]
    for k, v in tot.most_common(30):
        lines.append(f"| {v / T * 100:.2f}% | {v / 1e3:.1f} | {cnt[k]} | `{k}` |")
    stats = {"step_kernels": e - s, "step_device_us": T / 1e3,
             "owned_share": sum(owned.values()) / T, "nccl_share": sum(nccl.values()) / T,
             "owned": {k: v / T for k, v in owned.items()},
             "model_side_share": sum(model_side.values()) / T,
             "model_side": {k: v / T for k, v in model_side.items()}}
    return "\n".join(lines), stats


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--full")
    ap.add_argument("--launches")
    ap.add_argument("--tag", default="r1")
    ap.add_argument("--config", default="")
    ap.add_argument("--adamw-bytes", type=float, default=0.0)
    ap.add_argument("--acc-bytes", type=float, default=0.0)
    ap.add_argument("--acc-first-bytes", type=float, default=0.0)
    ap.add_argument("--acc-multi-bytes", type=float, default=0.0)
    ap.add_argument("--acc-multi-first-bytes", type=float, default=0.0)
    a = ap.parse_args()
    if a.full:
        algo = {}
        if a.adamw_bytes:
            algo["het_adamw"] = a.adamw_bytes
        if a.acc_bytes:
            algo["het_accumulate"] = a.acc_bytes
        if a.acc_first_bytes:
            algo["het_accumulate_first"] = a.acc_first_bytes
        if a.acc_multi_bytes:
            algo["het_accumulate_multi"] = a.acc_multi_bytes
        if a.acc_multi_first_bytes:
            algo["het_accumulate_multi_first"] = a.acc_multi_first_bytes
        summ = full_summary(a.full, algo, a.config)
        dst = HERE / "ncu_summary.json"
        prev = json.loads(dst.read_text()) if dst.exists() else {}
        prev.update(summ)
        dst.write_text(json.dumps(prev, indent=2, sort_keys=True) + "\n")
        print(json.dumps(summ, indent=2))
    if a.launches:
        table, stats = launch_shares(a.launches)
        (HERE / f"{a.tag}_launch_shares.md").write_text(
            f"# Launch list, one step ({a.config})\n\nSerialized cold-cache ncu "
            f"`gpu__time_duration.sum` per launch (compare shares, not absolutes).\n\n"
            f"```json\n{json.dumps(stats, indent=2)}\n```\n\n{table}\n")
        print(json.dumps(stats, indent=2))


if __name__ == "__main__":
    main()

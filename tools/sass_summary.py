#!/usr/bin/env python
"""Static evidence for the owned kernels of libhetstep.so (no GPU needed):
per kernel, registers / local memory (spills) from `cuobjdump -res-usage`,
and from `cuobjdump -sass` the global memory instructions by width
(LDG/STG .64 / .128 / 256-bit ENL2.256), the NVLS multimem instructions
(LDGMC = multimem.ld_reduce, STGMC... = multimem.st) and the system-scope
release/acquire of the fused collectives' barriers.

  python tools/sass_summary.py [--lib paper_2411_01075_b200/_lib/libhetstep.so] \
      [--out profiles/r2_sass_summary.md]
"""
import argparse
import collections
import re
import subprocess

OWNED = ("adamw", "accumulate", "pack", "embedding_grad", "fill", "gather_bf16",
         "symm_ag", "symm_rs", "symm_virtual", "status_copy", "epoch_update")


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True,
                         text=True).stdout.splitlines()
    return dict(zip(names, out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default="paper_2411_01075_b200/_lib/libhetstep.so")
    ap.add_argument("--out", default="profiles/r2_sass_summary.md")
    a = ap.parse_args()
    res = subprocess.run(["cuobjdump", "-res-usage", a.lib], capture_output=True,
                         text=True).stdout
    usage, cur = {}, None
    for line in res.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            cur = m.group(1)
        elif cur and "REG:" in line:
            usage[cur] = {k: int(v) for k, v in re.findall(r"(REG|STACK|LOCAL|SHARED):(\d+)", line)}
            cur = None
    sass = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True).stdout
    counts, cur = {}, None
    # every memory opcode with its full modifier string (LDG.E.EF.128, ST.E.128,
    # LDGMC.E.ADD.F32x4.RN.STRONG.SYS, STG.E.128.STRONG.SYS, ...)
    pat = re.compile(r"\b((?:LDGMC|LDG|STG|LDS|STS|LD|ST|RED|ATOM|MEMBAR|FENCE)"
                     r"(?![A-Za-z0-9])(?:\.[A-Za-z0-9_]+)*)")
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None or "/*" not in line:
            continue
        body = line.split("*/", 1)[-1].split(";")[0]
        for op in pat.findall(body):
            if op.startswith(("LDS", "STS")):
                continue                     # shared memory
            counts[cur][op] += 1
    names = sorted(set(usage) | set(counts))
    dm = demangle(names)
    rows = []
    for n in names:
        d = dm.get(n, n)
        short = d.replace("(anonymous namespace)::", "").replace("void ", "", 1)
        short = re.sub(r"\(.*", "", short)
        if not any(k in short for k in OWNED):
            continue
        u = usage.get(n, {})
        c = counts.get(n, {})
        mem = ", ".join(f"{k} {v}" for k, v in sorted(c.items()))
        rows.append(f"| `{short}` | {u.get('REG', '?')} | {u.get('LOCAL', '?')} | {mem} |")
    text = ["# Owned kernels: registers, spills, memory instructions (static, from SASS)", "",
            f"`python tools/sass_summary.py` on `{a.lib}` (sm_100a). LOCAL = bytes of local",
            "memory per thread (0: no spills). Opcode counts in the SASS, shared memory left",
            "out: `.128` / `.ENL2.256` = 16- / 32-byte accesses, `.EF` = evict-first;",
            "LDGMC = `multimem.ld_reduce` (NVLS switch reduction); `multimem.st` assembles to",
            "`STG.E.128.STRONG.SYS` on the multicast address; `LD.E` / `ST.E` = generic",
            "accesses (the fused collectives' peer-mapped NVLink loads / stores);",
            "`.STRONG.SYS` scalar LD/ST = the cross-rank barrier flags.", "",
            "| kernel | regs | local B | global / multimem / system-scope memory instructions |",
            "|---|---|---|---|"] + rows
    open(a.out, "w").write("\n".join(text) + "\n")
    print("\n".join(text))


if __name__ == "__main__":
    main()

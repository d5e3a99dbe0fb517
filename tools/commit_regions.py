#!/usr/bin/env python3
"""k_tick_commit time by code region: ncu per-instruction warp-stall samples (helper-warp
ring waits excluded) grouped by the CommitT member function / kernel section each source
line belongs to.  python tools/commit_regions.py REPORT.ncu-rep LIB.so"""
import collections
import csv
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_line_profile import line_table  # noqa: E402

SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2505_01968_b200", "csrc", "rapp_tick.cu")


def regions():
    """[(first line, name)] of CommitT's members and k_tick_commit's sections."""
    out = []
    for i, ln in enumerate(open(SRC).read().splitlines(), 1):
        m = re.match(r"\s+__device__ (?:static )?[\w:<>\s\*&]+?\b(\w+)\(", ln)
        if m and "inline" not in ln:
            out.append((i, m.group(1)))
        if "__global__" in ln:
            m = re.search(r"\b(k_\w+)\(", ln)
            out.append((i, m.group(1) if m else "kernel"))
        if "warp 0: the commit" in ln:
            out.append((i, "commit main loop"))
        if "every warp: the shared-memory cluster state back" in ln:
            out.append((i, "epilogue"))
        if "if (threadIdx.x >= 32) {" in ln:
            out.append((i, "helper warps"))
    return sorted(out)


def main(rep, lib):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    base = int(data[0]["Address"], 16)
    lo = line_table(lib, "k_tick_commit")
    regs = regions()

    def reg(line):
        m = re.match(r"rapp_tick\.cu:(\d+)", line or "")
        if not m:
            return (line or "?").split(":")[0]
        n = int(m.group(1))
        name = "?"
        for start, nm in regs:
            if start <= n:
                name = nm
        return name
    samp, inst = collections.Counter(), collections.Counter()
    for d in data:
        r = reg(lo.get(int(d["Address"], 16) - base, "?"))
        samp[r] += sum(float(d[c] or 0) for c in hdr if c.startswith("stall_")
                       and "Not Issued" not in c and c not in ("stall_sleep", "stall_barrier"))
        inst[r] += float(d["Instructions Executed"] or 0)
    skip = {"helper warps", "prefetch_of", "sm_30_intrinsics.hpp"}
    tot = sum(v for k, v in samp.items() if k not in skip) or 1
    print(f"{'region':28s} samples%  warp-instr   (helper-side regions listed last)")
    for k, v in samp.most_common():
        if k not in skip:
            print(f"{k:28s} {100 * v / tot:7.1f}  {inst[k]:10.0f}")
    for k in skip:
        print(f"{k:28s} {'-':>7s}  {inst[k]:10.0f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

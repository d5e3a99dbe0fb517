#!/usr/bin/env python3
"""Per-source-line profile of one kernel from an ncu report (build with -lineinfo):
warp-stall samples (sleep/barrier samples of idle helper warps excluded), warp
instructions executed and the dominant stall reason, aggregated through the nvdisasm line
table.

    python tools/ncu_line_profile.py REPORT.ncu-rep LIB.so KERNEL_SUBSTRING [top]"""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile

SKIP = ("stall_sleep", "stall_barrier")


def line_table(lib, kname):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp,
                   capture_output=True)
    line_of = {}
    for cb in glob.glob(os.path.join(tmp, "*.cubin")):
        dis = subprocess.run(["nvdisasm", "-g", "-c", cb], capture_output=True, text=True).stdout
        cur_fn, cur_line = None, None
        for ln in dis.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", ln)
            if m:
                cur_fn = m.group(1)
                continue
            m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
            if m:
                cur_line = f"{m.group(1)}:{m.group(2)}"
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
            if m and cur_fn and kname in cur_fn:
                line_of[int(m.group(1), 16)] = cur_line
    return line_of


def main(rep, lib, kname, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    base = int(data[0]["Address"], 16)
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    line_of = line_table(lib, kname)
    samp, inst = collections.Counter(), collections.Counter()
    why = collections.defaultdict(collections.Counter)
    for d in data:
        ln = line_of.get(int(d["Address"], 16) - base, "?")
        inst[ln] += float(d["Instructions Executed"] or 0)
        for c in stall_cols:
            if c in SKIP:
                continue
            v = float(d[c] or 0)
            samp[ln] += v
            why[ln][c[6:]] += v
    ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
    print(f"active samples {ts:.0f}, warp instructions {ti:.0f}")
    for line, s in samp.most_common(top):
        w = ", ".join(f"{k} {100 * v / max(1, s):.0f}%" for k, v in why[line].most_common(2))
        print(f"{100 * s / ts:5.1f}% samples {100 * inst[line] / ti:5.1f}% inst  {line:24s} {w}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)

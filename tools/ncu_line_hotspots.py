#!/usr/bin/env python3
"""Warp-stall samples of one kernel aggregated by CUDA source line.

    python tools/ncu_line_hotspots.py REPORT.ncu-rep LIB.so KERNEL_SUBSTRING [top]

Maps ncu's per-SASS-instruction samples (--page source --print-source=sass) to source
lines through the line table nvdisasm prints for the cubin (build with -lineinfo)."""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile


def main(rep, lib, kname, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
    base = int(data[0]["Address"], 16)
    samples = {int(d["Address"], 16) - base: float(d["Warp Stall Sampling (All Samples)"] or 0)
               for d in data}
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp,
                   capture_output=True)
    cubins = glob.glob(os.path.join(tmp, "*.cubin"))
    line_of = {}
    for cb in cubins:
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
    agg = collections.Counter()
    for off, s in samples.items():
        agg[line_of.get(off, "?")] += s
    tot = sum(agg.values()) or 1
    for line, s in agg.most_common(top):
        print(f"{100 * s / tot:5.1f}%  {line}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 25)

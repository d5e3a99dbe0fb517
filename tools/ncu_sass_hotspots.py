"""Summarise an ncu report's SASS source page: top instructions by warp-stall samples and
per-opcode instruction counts (helper for profiles/ summaries)."""
import collections
import csv
import subprocess
import sys


def sass_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def main(rep, top=30):
    rows = sass_rows(rep)
    tot = sum(float(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows) or 1
    ops = collections.Counter()
    for r in rows:
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        ops[op.split(".")[0]] += int(r["Thread Instructions Executed"] or 0)
    rows.sort(key=lambda r: -float(r["Warp Stall Sampling (All Samples)"] or 0))
    for r in rows[:top]:
        s = float(r["Warp Stall Sampling (All Samples)"] or 0)
        print(f"{100 * s / tot:5.1f}%  {r['Source'].strip()[:80]}")
    print("--- thread instructions by opcode ---")
    for op, n in ops.most_common(25):
        print(f"{op:12s} {n:,}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)

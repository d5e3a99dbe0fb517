#!/usr/bin/env python3
"""Aggregates an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel into the
profiles/ JSON form: launches, total µs and share of all profiled kernel time.

    python tools/ncu_launch_list.py LAUNCHES.csv "COMMAND" > profiles/rNN_launches_X.json
"""
import collections
import csv
import json
import sys


def main(path, command):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value",
                                             "Metric Unit"))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
             "second": 1e6, "s": 1e6}
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[name] += 1
    all_us = sum(tot.values()) or 1.0
    out = {"command": command,
           "note": "per-launch times are cold-cache and serialised; shares, not absolutes, "
                   "are comparable with the bench",
           "kernels": [{"kernel": k, "launches": cnt[k], "total_us": round(v, 1),
                        "share": round(v / all_us, 4)} for k, v in tot.most_common()]}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

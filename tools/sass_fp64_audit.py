#!/usr/bin/env python3
"""FP64 audit of librapp_b200.so's SASS: per kernel, DADD / DMUL / DFMA / MUFU.RCP64H counts
and where every DFMA sits.  Every reference expression is evaluated with individually
rounded operations (no contraction), so a DFMA may only appear
  * inside a correctly rounded IEEE division (__ddiv_rn / '/' expands to MUFU.RCP64H plus a
    DFMA Newton/correction sequence — the division itself is exact-rounded), or
  * in the exact-by-construction fma(k, h, a0) of a uniform axis's node (rapp_stream.cu
    locate_fast<UNIFORM>, k*h + a0 exactly representable).
A DFMA outside a division window is reported with its source line (build with -lineinfo).

    python tools/sass_fp64_audit.py [LIB.so]"""
import collections
import re
import subprocess
import sys

WINDOW = 40  # instructions around a MUFU.RCP64H that belong to its division expansion


def main(lib):
    dis = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    fn, ins = None, collections.OrderedDict()
    for ln in dis.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            fn = m.group(1)
            ins.setdefault(fn, [])
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4}\*/\s+(.*?);", ln)
        if m and fn:
            ins[fn].append(m.group(1).strip())
    tot = collections.Counter()
    print(f"{'kernel':70s} DADD DMUL DFMA RCP64H DFMA-outside-div")
    for fn, lst in ins.items():
        ops = [re.sub(r"^@!?U?P\w+\s+", "", x).split()[0] if x else "" for x in lst]
        c = collections.Counter(o.split(".")[0] for o in ops)
        rcp = [i for i, o in enumerate(ops) if o.startswith("MUFU.RCP64H")]
        rets = [i for i, o in enumerate(ops) if o.startswith("RET")]
        exits = [i for i, o in enumerate(ops) if o.startswith("EXIT")]

        def in_subroutine(i):
            # the division slow path (CUDA's out-of-line __internal ddiv) is a subroutine
            # placed after the kernel body: the next RET comes before any EXIT
            r = next((x for x in rets if x > i), None)
            e = next((x for x in exits if x > i), None)
            return r is not None and (e is None or r < e)
        outside = [i for i, o in enumerate(ops) if o.startswith("DFMA")
                   and not any(abs(i - r) <= WINDOW for r in rcp) and not in_subroutine(i)]
        if c["DADD"] + c["DMUL"] + c["DFMA"] == 0:
            continue
        name = fn if len(fn) <= 70 else fn[:67] + "..."
        print(f"{name:70s} {c['DADD']:4d} {c['DMUL']:4d} {c['DFMA']:4d} {len(rcp):6d} "
              f"{len(outside):6d}")
        for k in ("DADD", "DMUL", "DFMA"):
            tot[k] += c[k]
        tot["RCP64H"] += len(rcp)
        tot["outside"] += len(outside)
    print(f"{'total':70s} {tot['DADD']:4d} {tot['DMUL']:4d} {tot['DFMA']:4d} "
          f"{tot['RCP64H']:6d} {tot['outside']:6d}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "paper_2505_01968_b200/librapp_b200.so")

#!/usr/bin/env python3
"""Summarise one kernel of an ncu --set full report into a JSON record for profiles/.

    python tools/ncu_summary.py REPORT.ncu-rep [--units N] [--unit-name predictions]

Prints duration, DRAM bytes (read/write, per unit), achieved DRAM GB/s, L1/L2/issue
utilisation, FP64-pipe activity and the top warp-stall reasons.
"""
import argparse
import csv
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_pct",
    "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed": "l1_wavefront_pct",
    "lts__t_sectors.sum.pct_of_peak_sustained_elapsed": "l2_sector_pct",
    "sm__inst_executed.sum.pct_of_peak_sustained_elapsed": "issue_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma_thread_inst",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd_thread_inst",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul_thread_inst",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__ops_path_tensor_src_bf16_dst_fp32.sum.pct_of_peak_sustained_elapsed": "tensor_bf16_ops_pct",
    "smsp__sass_inst_executed_op_utcmma.sum": "utcmma_inst",
}
UNITS = {"dram__bytes_read.sum": 1, "dram__bytes_write.sum": 1}


def to_bytes(val, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
             "GB": 1e9}.get(unit, 1)
    return float(val) * scale


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--units", type=float, default=None)
    ap.add_argument("--unit-name", default="units")
    ap.add_argument("--kernel-index", type=int, default=0)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2 + a.kernel_index]
    rec = {"report": a.report, "kernel": vals[hdr.index("Kernel Name")][:160]}
    stalls = {}
    for k, u, v in zip(hdr, units, vals):
        if k in KEYS:
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            if k in UNITS:
                x = to_bytes(x, u)
            if k == "gpu__time_duration.sum" and u == "ms":
                x *= 1000.0
            if k == "gpu__time_duration.sum" and u == "ns":
                x /= 1000.0
            rec[KEYS[k]] = x
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stalls[k[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(v)
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    rec["stall_top"] = {k: round(100 * v / tot, 1) for k, v in
                        sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
    if "dram_read_bytes" in rec and "duration_us" in rec:
        tb = rec["dram_read_bytes"] + rec["dram_write_bytes"]
        rec["dram_bytes"] = tb
        rec["dram_gbs"] = tb / (rec["duration_us"] * 1e-6) / 1e9
        if a.units:
            rec[a.unit_name] = a.units
            rec[f"dram_bytes_per_{a.unit_name}"] = tb / a.units
            rec[f"{a.unit_name}_per_s"] = a.units / (rec["duration_us"] * 1e-6)
    print(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main()

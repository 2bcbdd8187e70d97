"""Summarise an ncu --set full report (read here, no GPU needed).

usage: python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep [--json out.json] [--md out.md] [--tag kind]
Prints the metrics the roofline discussion in DESIGN.md uses, per profiled kernel.
"""
import argparse
import csv
import io
import json
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/SMEM % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe % active"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 inst % of peak"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA sub-pipe % active"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs, blocks)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem ld wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "smem st wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("lts__t_bytes.sum", "L2 bytes"),
]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
        for key, label in METRICS:
            if key in hdr:
                i = hdr.index(key)
                d[key] = (r[i], units[i])
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--json")
    ap.add_argument("--md")
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    res = load(a.rep)
    lines = []
    for d in res:
        lines.append(f"### {d['kernel'][:120]}")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for key, label in METRICS:
            if key in d:
                v, u = d[key]
                lines.append(f"| {label} (`{key}`) | {v} {u} |")
        lines.append("")
    md = "\n".join(lines)
    print(md)
    if a.md:
        with open(a.md, "w") as f:
            f.write(md)
    if a.json:
        with open(a.json, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

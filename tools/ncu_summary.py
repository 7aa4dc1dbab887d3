#!/usr/bin/env python
"""Summarise an .ncu-rep (read offline with `ncu -i`) into a short text file for profiles/."""
import csv
import subprocess
import sys
from collections import Counter

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum",
        "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_barrier",
        "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
        "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
        "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_selected",
        "smsp__pcsamp_warps_issue_stalled_not_selected", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg"]


def run(args):
    return subprocess.run(args, capture_output=True, text=True).stdout


def main(rep, out, note=""):
    raw = list(csv.reader(run(["ncu", "-i", rep, "--page", "raw", "--csv"]).splitlines()))
    hdr, units = raw[0], raw[1]
    lines = [f"# {rep}", f"# {note}"]
    for r in raw[2:]:
        lines.append("kernel: " + r[hdr.index("Kernel Name")][:110])
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"  {k} = {r[i]} {units[i]}")
    src = list(csv.reader(run(["ncu", "-i", rep, "--page", "source", "--csv"]).splitlines()))
    kern, h, c, ce, tot = 0, None, Counter(), Counter(), 0
    for r in src:
        if r and r[0] == "Kernel Name":
            kern += 1
            continue
        if r and r[0] == "Address":
            h = {x: i for i, x in enumerate(r)}
            continue
        if kern == 1 and h and len(r) > 5:
            toks = r[h["Source"]].split()
            op = toks[1] if toks[0].startswith("@") else toks[0]
            op = op.split(".")[0]
            s = int(r[h["# Samples"]])
            c[op] += s
            ce[op] += int(r[h["Instructions Executed"]])
            tot += s
    lines.append("stall samples by opcode (first captured launch): opcode samples share executed_warp_instr")
    for k, v in c.most_common(16):
        lines.append(f"  {k} {v} {100 * v / max(tot, 1):.1f}% {ce[k]}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], " ".join(sys.argv[3:]))

"""Summarise an ncu report: key metrics + top source lines by instructions/stalls.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--lines 30]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio"]


def run(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    nlines = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    rows = list(csv.reader(io.StringIO(run(rep, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print("kernel:", d.get("Kernel Name", "?")[:120])
        for k in KEYS:
            if k in d:
                print(f"  {k:80s} {d[k]:>16s} {units[hdr.index(k)]}")
    src = list(csv.reader(io.StringIO(run(rep, "--page", "source", "--csv",
                                          "--print-source=cuda,sass"))))
    out, fname, h = [], None, None
    for r in src:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            h = r
            continue
        if h and len(r) == len(h) and r[2] == "-":
            try:
                ie, st = int(r[7]), int(r[4])
            except ValueError:
                continue
            if ie:
                out.append((ie, st, fname, r[0], r[1][:90]))
    tot = sum(o[0] for o in out) or 1
    tst = sum(o[1] for o in out) or 1
    print(f"\ntop source lines (of {tot} warp instructions, {tst} stall samples)")
    for o in sorted(out, reverse=True)[:nlines]:
        print(f"{o[0] / tot * 100:5.1f}% inst {o[1] / tst * 100:5.1f}% stall  {o[2]}:{o[3]}  {o[4]}")


if __name__ == "__main__":
    main()

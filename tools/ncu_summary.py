#!/usr/bin/env python3
"""Summarise an ncu report (speed of light, occupancy, DRAM traffic, stall
reasons, top source lines) into plain text for profiles/, one block per profiled
kernel launch.  Usage: ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEEP = {"Duration", "DRAM Throughput", "Compute (SM) Throughput", "Memory Throughput", "Issue Slots Busy",
        "Executed Ipc Active", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Achieved Active Warps Per SM", "Eligible Warps Per Scheduler", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "Executed Instructions",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
        "Branch Efficiency"}
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum",
       "sm__inst_issued.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
       "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
       "smsp__pcsamp_warps_issue_stalled_not_selected", "smsp__pcsamp_warps_issue_stalled_selected",
       "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_mio_throttle"]


def run(args):
    return subprocess.run(["ncu", "-i", sys.argv[1]] + args, capture_output=True, text=True).stdout


def main():
    det = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
    hdr = det[0]
    raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
    rhdr, runits, rrows = raw[0], raw[1], raw[2:]
    ids = []
    for row in det[1:]:
        d = dict(zip(hdr, row))
        if d["ID"] not in ids:
            ids.append(d["ID"])
    for n, kid in enumerate(ids):
        rows = [dict(zip(hdr, r)) for r in det[1:] if r[0] == kid]
        print(f"######## launch {kid}: {rows[0]['Kernel Name']}")
        print("== details")
        for d in rows:
            if d.get("Metric Name") in KEEP:
                print(f"  {d['Metric Name']:40s} {d['Metric Value']:>16s} {d['Metric Unit']}")
        if n < len(rrows):
            d = dict(zip(rhdr, rrows[n]))
            u = dict(zip(rhdr, runits))
            print("== dram / kernel")
            for k in RAW:
                print(f"  {k:55s} {d.get(k)} {u.get(k, '')}")
            st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", "") or 0)
                  for k, v in d.items()
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
            tot = sum(st.values()) or 1
            print("== stall samples (share)")
            for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:10]:
                print(f"  {k:30s} {100 * v / tot:5.1f}%")
        src = list(csv.reader(io.StringIO(run(["--page", "source", "--csv", "--print-source=cuda,sass",
                                                "--launch-skip", str(n), "--launch-count", "1"]))))
        cur, out, hd = None, [], None
        for r in src:
            if r and r[0] == "File Path":
                cur = r[1].split("/")[-1]
                continue
            if r and r[0] == "Line No":
                hd = r
                continue
            if hd and len(r) >= 10 and r[0] and r[2] == "-":
                try:
                    out.append((cur, int(r[0]), int(r[7]), int(r[4]), r[1][:80]))
                except ValueError:
                    pass
        ti = sum(o[2] for o in out) or 1
        ts = sum(o[3] for o in out) or 1
        print("== top source lines by stall samples (file line: %inst %stall source)")
        for o in sorted(out, key=lambda o: -o[3])[:20]:
            print(f"  {o[0][:16]:16s} {o[1]:4d} {100 * o[2] / ti:5.1f}% {100 * o[3] / ts:5.1f}%  {o[4]}")
        print()


if __name__ == "__main__":
    main()

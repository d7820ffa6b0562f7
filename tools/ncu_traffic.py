#!/usr/bin/env python3
"""Per-kernel DRAM bytes, executed warp instructions, issue / pipe utilisation
and duration of an ncu report (one launch of every m3e kernel of one bench step)
-> profiles/<round>_bench_traffic.json, the file bench.py reads for
roofline.traffic and roofline.kernels (only when its source_hash matches the
CUDA sources bench.py runs).

Capture (one GPU, metrics only, the step after bench.py's 3 warm-up steps):
  ncu --kernel-name-base demangled -k regex:m3e:: -s 27 -c 9 --clock-control none \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,\
sm__inst_issued.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,\
sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,\
sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,launch__registers_per_thread \
      -o rep python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-phys
Usage: ncu_traffic.py rep.ncu-rep out.json "<command line of the capture>" [workload frames seed]
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
PIPES = {"issue_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
         "pipe_alu_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
         "pipe_fma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
         "pipe_xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
         "pipe_lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
         "registers": "launch__registers_per_thread"}


def short_name(name: str) -> str:
    name = name.replace("void ", "").strip()
    if "filter_kernel<5" in name or "filter_kernel<(int)5" in name:
        return "m3e::filter_kernel<SELECT_C, BIG=false>"
    if "filter_kernel<0" in name or "filter_kernel<(int)0" in name:
        big = "true" if ("true" in name or ", 1>" in name) else "false"
        return f"m3e::filter_kernel<FULL, BIG={big}>"
    if "fit_kernel<" in name:   # fit_kernel<BIG>: the phase-I variant is bench.py's "m3e::fit_kernel"
        big = "true" in name or "<1>" in name or "(bool)1" in name
        return "m3e::fit_kernel<BIG>" if big else "m3e::fit_kernel"
    base = name.split("(")[0]
    return base if base.startswith("m3e::") else "m3e::" + base


def main():
    rep, out_path, source = sys.argv[1], sys.argv[2], sys.argv[3]
    workload, frames, seed = (sys.argv[4], int(sys.argv[5]), int(sys.argv[6])) if len(sys.argv) > 6 else \
        ("phase1_sig", 15625000, 20220623)
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    res = {}
    for r in data:
        short = short_name(r[ix["Kernel Name"]])
        val = lambda k: float(r[ix[k]].replace(",", ""))
        t_unit = units[ix["gpu__time_duration.sum"]]
        e = {
            "dram_read_bytes": round(val("dram__bytes_read.sum") * SCALE[units[ix["dram__bytes_read.sum"]]]),
            "dram_write_bytes": round(val("dram__bytes_write.sum") * SCALE[units[ix["dram__bytes_write.sum"]]]),
            "inst_executed": int(val("smsp__inst_executed.sum")),
            "ms_under_ncu": val("gpu__time_duration.sum") * {"ms": 1.0, "us": 1e-3, "ns": 1e-6}[t_unit],
        }
        for k, m in PIPES.items():
            if m in ix and r[ix[m]] not in ("", "n/a"):
                e[k] = val(m)
        res[short] = e
    import bench
    with open(out_path, "w") as fh:
        json.dump({"workload": workload, "frames": frames, "seed": seed, "source_hash": bench.kernel_source_hash(),
                   "kernels": res, "source": source}, fh, indent=1)
    for k, v in res.items():
        print(k, v)


if __name__ == "__main__":
    main()

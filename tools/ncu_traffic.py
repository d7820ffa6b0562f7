#!/usr/bin/env python3
"""Per-kernel DRAM bytes, executed warp instructions and duration of an ncu
report (one launch per kernel) -> profiles/<round>_bench_traffic.json, the file
bench.py reads for roofline.traffic and roofline.issue.
Usage: ncu_traffic.py report.ncu-rep out.json "<command line of the capture>" """
import csv
import io
import json
import subprocess
import sys

SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def main():
    rep, out_path, source = sys.argv[1], sys.argv[2], sys.argv[3]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    res = {}
    for r in data:
        name = r[ix["Kernel Name"]]
        short = "m3e::" + name.split("(")[0].replace("void ", "").strip()
        if "filter_kernel<5" in name:
            short = "m3e::filter_kernel<SELECT_C, BIG=false>"
        elif "filter_kernel<0" in name:
            short = "m3e::filter_kernel<FULL, BIG=false> (spilled warp-batches)"
        val = lambda k: float(r[ix[k]].replace(",", ""))
        t_unit = units[ix["gpu__time_duration.sum"]]
        res[short] = {
            "dram_read_bytes": round(val("dram__bytes_read.sum") * SCALE[units[ix["dram__bytes_read.sum"]]]),
            "dram_write_bytes": round(val("dram__bytes_write.sum") * SCALE[units[ix["dram__bytes_write.sum"]]]),
            "inst_executed": int(val("smsp__inst_executed.sum")),
            "ms_under_ncu": val("gpu__time_duration.sum") * {"ms": 1.0, "us": 1e-3, "ns": 1e-6}[t_unit],
        }
    with open(out_path, "w") as fh:
        json.dump({"workload": "phase1_sig", "frames": 15625000, "seed": 20220623, "kernels": res, "source": source},
                  fh, indent=1)
    for k, v in res.items():
        print(k, v)


if __name__ == "__main__":
    main()

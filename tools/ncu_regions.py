#!/usr/bin/env python3
"""Executed-instruction and stall-sample shares per device function / kernel
stage from an ncu report's source page (needs -lineinfo)."""
import collections
import csv
import io
import os
import subprocess
import sys

SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2206_11535_b200", "csrc")


def region(files, f, line):
    src = files.get(f)
    if src is None:
        return f
    for k in range(line - 1, -1, -1):
        t = src[k]
        if "// ----" in t and ":" in t:
            return f"{f}:{t.strip().strip('/- ')[:40]}"
        if (t.startswith(("M3E_HD", "__device__", "static __device__", "__global__", "template <class"))
                and "(" in t):
            return f"{f}:{t.split('(')[0].split()[-1]}"
    return f + ":?"


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    files = {}
    for fn in ("m3e_device.cuh", "m3e_kernels.cu"):
        files[fn] = open(os.path.join(SRC, fn)).read().split("\n")
    cur, hdr = None, None
    ins, st = collections.Counter(), collections.Counter()
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "File Path":
            cur = os.path.basename(r[1])
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) >= 10 and r[0] and r[2] == "-":
            try:
                key = region(files, cur, int(r[0]))
                ins[key] += int(r[7])
                st[key] += int(r[4])
            except ValueError:
                pass
    ti, ts = sum(ins.values()) or 1, sum(st.values()) or 1
    print(f"executed warp instructions: {ti}")
    for k, v in ins.most_common(30):
        print(f"  {100 * v / ti:5.1f}% inst  {100 * st[k] / ts:5.1f}% stall  {k}")


if __name__ == "__main__":
    main()

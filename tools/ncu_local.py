#!/usr/bin/env python3
"""Per-source-line share of one ncu column (default: local-memory L2 sectors)
for one kernel of an ncu report, mapping SASS addresses back to CUDA lines with
nvdisasm -g of the library's cubins.
Usage: ncu_local.py report.ncu-rep lib.so kernel_symbol_substring launch_skip [column] [top]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main():
    rep, lib, pat, skip = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
    col = sys.argv[5] if len(sys.argv) > 5 else "L2 Theoretical Sectors Local"
    top = int(sys.argv[6]) if len(sys.argv) > 6 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "--launch-skip",
                          str(skip), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    iA, iC = hdr.index("Address"), hdr.index(col)
    data = {}
    for r in rows:
        if len(r) == len(hdr) and r[iA].startswith("0x"):
            data[int(r[iA], 16)] = float(r[iC] or 0)
    base = min(data)
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
        text = ""
        for fn in sorted(os.listdir(d)):
            if fn.endswith(".cubin"):
                text += subprocess.run(["nvdisasm", "-g", os.path.join(d, fn)], capture_output=True,
                                       text=True).stdout
    on, cur, amap = False, None, {}
    for line in text.split("\n"):
        if line.startswith("//--------------------- .text."):
            on = pat in line
            continue
        if not on:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = os.path.basename(m.group(1)) + ":" + m.group(2)
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
        if m:
            amap[int(m.group(1), 16)] = cur
    by = collections.Counter()
    for a, v in data.items():
        by[amap.get(a - base, "?")] += v
    tot = sum(by.values()) or 1.0
    print(f"{col}: total {tot:.4g}")
    for l, v in by.most_common(top):
        print(f"  {v / tot * 100:5.1f}%  {l}")


if __name__ == "__main__":
    main()

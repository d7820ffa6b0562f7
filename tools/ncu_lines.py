#!/usr/bin/env python3
"""Per-source-line executed warp instructions and stall samples of ONE kernel
launch of an ncu report (source page, needs -lineinfo), sorted by instructions.
Usage: ncu_lines.py report.ncu-rep launch_index [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep, k = sys.argv[1], int(sys.argv[2])
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                          "--launch-skip", str(k), "--launch-count", "1"], capture_output=True, text=True).stdout
    cur, hdr, rows = None, None, []
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] in ("File Name", "File Path"):
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) > 7 and r[0] and r[2] == "-":
            try:
                ins, st = int(r[7]), int(r[4])
            except ValueError:
                continue
            if ins or st:
                rows.append((ins, st, cur, r[0], r[1].strip()[:90]))
    ti = sum(r[0] for r in rows) or 1
    ts = sum(r[1] for r in rows) or 1
    print(f"executed warp instructions: {ti}")
    for ins, st, f, ln, src in sorted(rows, reverse=True)[:top]:
        print(f"{100 * ins / ti:5.1f}% {100 * st / ts:5.1f}%  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Static SASS evidence for the design claims (cuobjdump -sass of the built
library): per kernel, the count of the opcodes that prove TMA bulk copies
(UBLKCP, UBLKPF = cp.async.bulk[.prefetch]), async copies (LDGSTS), mbarriers
(SYNCS), packed fp32 (FFMA2 / FMUL2 / FADD2), MUFU, shared / global / local
memory and fp64, plus one example line of each proof opcode.
Usage: sass_summary.py lib.so > profiles/<round>_sass_summary.txt"""
import collections
import re
import subprocess
import sys

KEYS = ["UBLKCP", "UBLKPF", "LDGSTS", "SYNCS", "FFMA2", "FMUL2", "FADD2", "MUFU", "LDS", "STS", "LDG", "STG", "LD",
        "ST", "LDL", "STL", "DFMA", "DADD", "DMUL"]
PROOF = ["UBLKCP", "UBLKPF", "LDGSTS", "SYNCS", "FFMA2", "FMUL2", "FADD2"]


def main():
    txt = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
    print(f"# cuobjdump -sass {sys.argv[1]}")
    for f in re.split(r"\n\s*Function : ", txt)[1:]:
        name = f.split("\n", 1)[0].strip()
        ops, ex = collections.Counter(), {}
        for line in f.splitlines():
            m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?\s*(.*?);", line)
            if not m:
                continue
            op = m.group(2)
            ops[op] += 1
            if op in PROOF and op not in ex:
                ex[op] = (op + (m.group(3) or "") + " " + m.group(4)).strip()
        print(f"\n== {name}: {sum(ops.values())} instructions")
        print("   " + ", ".join(f"{k} {ops[k]}" for k in KEYS if ops[k]))
        for op, line in ex.items():
            print(f"   e.g. {line}")


if __name__ == "__main__":
    main()

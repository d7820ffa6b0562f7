#!/usr/bin/env python3
"""Static SASS instruction count per CUDA source line of one kernel
(nvdisasm -g on the cubins of a shared library): code-size budget tool.
Usage: sass_lines.py lib.so kernel_symbol_substring [top]"""
import collections
import os
import re
import subprocess
import sys
import tempfile


def main():
    lib, pat = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
        text = ""
        for fn in sorted(os.listdir(d)):
            if fn.endswith(".cubin"):
                text += subprocess.run(["nvdisasm", "-g", os.path.join(d, fn)], capture_output=True,
                                       text=True).stdout
    cnt, cur, on, src = collections.Counter(), None, False, {}
    for line in text.split("\n"):
        if line.startswith("//--------------------- .text."):
            on = pat in line
            continue
        if not on:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (m.group(1), int(m.group(2)))
            continue
        if re.search(r"/\*[0-9a-f]{4,}\*/", line) and cur:
            cnt[cur] += 1
    tot = sum(cnt.values())
    print(f"{tot} instructions in functions matching {pat!r}")
    for (f, l), c in cnt.most_common(top):
        if f not in src:
            try:
                src[f] = open(f).read().split("\n")
            except OSError:
                src[f] = []
        t = src[f][l - 1].strip()[:80] if l - 1 < len(src[f]) else ""
        print(f"{c:5d} {os.path.basename(f)}:{l} {t}")


if __name__ == "__main__":
    main()

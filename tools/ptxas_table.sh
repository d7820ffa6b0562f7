#!/bin/bash
# registers / spills / stack per kernel entry of libm3e (ptxas -v), one line each
cd "$(dirname "$0")/.." && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Iinclude -Ipaper_2206_11535_b200/csrc -c -o /tmp/m3e_k.o paper_2206_11535_b200/csrc/m3e_kernels.cu -Xptxas -v 2>&1 |
awk '/Compiling entry function/ {match($0, /_Z[^'"'"']*/); name=substr($0, RSTART, RLENGTH); getline; getline; sp=$0; getline;
     cmd="c++filt " name; cmd | getline dn; close(cmd); sub(/\(m3e::KArgs\)/, "", dn);
     match($0, /Used [0-9]+ registers/); printf "%-46s %-18s %s\n", dn, substr($0, RSTART+5, RLENGTH-5), sp}'

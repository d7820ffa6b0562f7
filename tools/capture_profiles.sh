#!/bin/bash
# One GPU call that regenerates the judged evidence under profiles/ for round $1
# (default r02): the ncu launch list of the bench command, the per-kernel
# counters bench.py reads (source-hashed), the bench line that reads them, full ncu summaries of the
# fit and selection kernels, and the SASS summary.  Run on the GPU box:
#   gpurun -- 'bash tools/capture_profiles.sh r02'
R=${1:-r02}
O=gpurun_out/$R
mkdir -p $O
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-phys > $O/launches.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,launch__registers_per_thread
ncu --kernel-name-base demangled -k regex:m3e:: -s 27 -c 9 --clock-control none --metrics $M -o $O/traffic \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-phys > $O/traffic.log 2>&1
python tools/ncu_traffic.py $O/traffic.ncu-rep $O/${R}_bench_traffic.json \
    "ncu --metrics <see tools/capture_profiles.sh> python bench.py --steps 1 --warmup 3 (the step after the warm-up)" > $O/traffic.txt 2>&1
# the bench line reads the counters of these very sources (this box's copy of profiles/).
# Cross-check only: right after the ncu passes the step measured 8.70 ms against 8.62
# on a fresh box (selection 3.78 vs 3.70 ms); the committed bench line is taken in a
# separate call once the counters are committed (python bench.py on a fresh box).
cp $O/${R}_bench_traffic.json profiles/
python bench.py > $O/bench_line_after_ncu.json 2> $O/bench_line.err
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"fit_kernel|filter_kernel" \
    -s 9 -c 2 -o $O/full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-phys > $O/full.log 2>&1
python tools/ncu_summary.py $O/full.ncu-rep > $O/${R}_bench_ncu_full.txt 2>&1
python bench.py --workload phase2_stress --frames 1000000 > $O/phase2_line.json 2> $O/phase2_line.err
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:filter_kernel \
    -s 6 -c 1 -o $O/p2 python bench.py --workload phase2_stress --frames 1000000 --steps 1 --warmup 3 --no-e2e --no-cpu --no-phys > $O/p2.log 2>&1
python tools/ncu_summary.py $O/p2.ncu-rep > $O/${R}_phase2_ncu.txt 2>&1
python bench.py --workload phase1_bg --frames 10000 --no-cpu > $O/configs1_line.json 2> $O/configs1.err
python bench.py --workload phase1_sig --frames 1000000 --no-cpu > $O/configs2_line.json 2> $O/configs2.err
echo done

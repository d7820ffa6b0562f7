#!/bin/bash
# Regenerates profiles/<round>_sanitizer.txt on the GPU box (one GPU):
#   gpurun -- 'bash tools/sanitize_all.sh r02'
R=${1:-r02}
O=gpurun_out/${R}_sanitizer.txt
: > $O
run() {   # header, tool, then the sanitize_run.py arguments
    echo "# compute-sanitizer $2, $1" >> $O
    compute-sanitizer --tool $2 python tools/sanitize_run.py "${@:3}" >> $O 2>&1
    echo "exit=$?" >> $O
}
run "split path: phase1_sig 20000, signal_only 3000, phase2_stress 300, single_frame 1, host path 5000" memcheck split
run "fused path: phase1_sig 20000, signal_only 3000, phase2_stress 300, single_frame 1, host path 5000" memcheck fused
run "spill path: phase1_sig 20000, signal_only 3000, phase2_stress 300, single_frame 1, host path 5000" memcheck spill
run "(shared-memory hazards), split path: phase1_sig 3000, phase2_stress 40" racecheck split phase1_sig:3000 phase2_stress:40
run "split path: phase1_sig 3000, phase2_stress 40" synccheck split phase1_sig:3000 phase2_stress:40

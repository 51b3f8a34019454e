#!/bin/bash
# Round profile (GPU box): C3 launch list of one timed step + ncu --set full of the dominant
# kernel's launches in that step (and one shade / backward launch).  Scratch in gpurun_out/;
# tools/ncu_summary.py turns it into profiles/.   Usage: tools/profile_round.sh TAG
T=${1:-r01}
B="python bench.py --config C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
export BENCH_NO_CLOCKS=1
$B > gpurun_out/${T}_b0.log 2>&1 || { echo "bench failed"; tail -5 gpurun_out/${T}_b0.log; exit 1; }
tail -1 gpurun_out/${T}_b0.log > gpurun_out/${T}_bench_1step.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $B > gpurun_out/${T}_ncu0.log 2>&1
echo "launch list rc=$?"
# the timed step's 4 traversal launches: 4 (target render) + 3 x 4 (warm-up) = 16 before it
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_traverse_level -s 16 -c 4 -o gpurun_out/${T}_traverse $B > gpurun_out/${T}_ncu1.log 2>&1
echo "ncu traverse rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_shade_level -s 22 -c 1 -o gpurun_out/${T}_shade $B > gpurun_out/${T}_ncu2.log 2>&1
echo "ncu shade rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_backward_level -s 16 -c 1 -o gpurun_out/${T}_bwd $B > gpurun_out/${T}_ncu3.log 2>&1
echo "ncu bwd rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_trace_primary -s 4 -c 1 -o gpurun_out/${T}_primary $B > gpurun_out/${T}_ncu4.log 2>&1
echo "ncu primary rc=$?"

#!/bin/bash
# ncu captures of the C3V (volumetric env) shade and backward (level-1 launches of the timed step)
T=${1:-c3v}
B="python bench.py --config C3V --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
export BENCH_NO_CLOCKS=1
$B > gpurun_out/${T}_b0.log 2>&1 || { echo "bench failed"; tail -5 gpurun_out/${T}_b0.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_backward_level -s 19 -c 1 -o gpurun_out/${T}_bwd $B > gpurun_out/${T}_ncu_bwd.log 2>&1; echo "ncu bwd rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_shade_level -s 21 -c 1 -o gpurun_out/${T}_shade $B > gpurun_out/${T}_ncu_shade.log 2>&1; echo "ncu shade rc=$?"

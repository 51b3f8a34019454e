#!/bin/bash
# ncu captures of the C4 (sigma-grid) backward and shade kernels.  Usage: tools/ncu_c4.sh TAG
T=${1:-c4}
B="python bench.py --config C4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
export BENCH_NO_CLOCKS=1
$B > gpurun_out/${T}_b0.log 2>&1 || { echo "bench failed"; tail -5 gpurun_out/${T}_b0.log; exit 1; }
tail -1 gpurun_out/${T}_b0.log | cut -c1-400
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_backward_level -s 23 -c 1 -o gpurun_out/${T}_bwd $B > gpurun_out/${T}_ncu_bwd.log 2>&1; echo "ncu bwd rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_shade_level -s 32 -c 1 -o gpurun_out/${T}_shade $B > gpurun_out/${T}_ncu_shade.log 2>&1; echo "ncu shade rc=$?"

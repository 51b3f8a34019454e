#!/bin/bash
# GPU-box round: parity tests, bench, launch list and ncu captures (scratch under gpurun_out/).
python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 900 > gpurun_out/gpu.log 2>&1; tail -4 gpurun_out/gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log
B="python bench.py --config C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
if [ "${NCU:-1}" = "1" ]; then
$B > gpurun_out/b1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu1.log 2>&1
echo "launch list rc=$?"
$B > gpurun_out/b2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_traverse_level -s 16 -c 1 -o gpurun_out/prof_traverse $B > gpurun_out/ncu2.log 2>&1
echo "ncu traverse rc=$?"
$B > gpurun_out/b3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_backward_level -s 15 -c 1 -o gpurun_out/prof_bwd $B > gpurun_out/ncu3.log 2>&1
echo "ncu bwd rc=$?"
$B > gpurun_out/b4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_shade_level -s 20 -c 1 -o gpurun_out/prof_shade $B > gpurun_out/ncu4.log 2>&1
echo "ncu shade rc=$?"
fi

python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 900 > gpurun_out/gpu2.log 2>&1; tail -6 gpurun_out/gpu2.log
B="python bench.py --config C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/b1.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu1.log 2>&1
echo "launch list rc=$?"
$B > gpurun_out/b2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_trace_level -s 16 -c 1 -o gpurun_out/prof_trace $B > gpurun_out/ncu2.log 2>&1
echo "ncu trace rc=$?"
$B > gpurun_out/b3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_backward_level -s 20 -c 1 -o gpurun_out/prof_bwd $B > gpurun_out/ncu3.log 2>&1
echo "ncu bwd rc=$?"
tail -2 gpurun_out/ncu2.log

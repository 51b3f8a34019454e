#!/bin/bash
# GPU box: parity tests + smoke + a short C3 bench (scratch output in gpurun_out/)
mkdir -p gpurun_out
export PARITY_REPORT=gpurun_out/parity_report.jsonl
rm -f $PARITY_REPORT
timeout ${PT:-2400} python -m pytest tests/${TESTS:-test_gpu_parity.py} -q -m gpu --timeout 1200 ${PYARGS} > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
if [ -n "$BENCH" ]; then
  timeout 600 python bench.py --config ${BENCH} --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${BENCH}.json 2> gpurun_out/bench_${BENCH}.err
  echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_${BENCH}.json; tail -3 gpurun_out/bench_${BENCH}.err
fi

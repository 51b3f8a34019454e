#!/bin/bash
# GPU box: the bench line of every config (device + e2e + cpu_baseline) into gpurun_out/r02_bench_*.json
mkdir -p gpurun_out
for c in C1 C2 C3 C4 C5 C4H C3V; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err
  echo "$c rc=$? $(python -c "import json;d=json.load(open('gpurun_out/r02_bench_$c.json'));print(d['value'],d['e2e']['value'] if d.get('e2e') else None,d['ms_per_step'],(d.get('cpu_baseline') or {}).get('value'))" 2>/dev/null)"
done
timeout 900 python bench.py --mode infer --steps ${STEPS:-10} --warmup 3 > gpurun_out/r02_bench_C3R_infer.json 2> gpurun_out/r02_bench_C3R.err
echo "C3R infer rc=$?"
timeout 600 python bench.py --batch 5000 --steps 200 --warmup 5 > gpurun_out/r02_bench_C3_batch5000.json 2> gpurun_out/r02_bench_batch.err
echo "batch rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
echo "reference rc=$?"

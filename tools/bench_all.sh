#!/bin/bash
# every bench workload once (GPU box); lines into gpurun_out/bench_<cfg>.json
python bench.py > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; tail -1 gpurun_out/bench_C3.json | cut -c1-150
for c in C2 C4 C5 C4H C3V; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  tail -1 gpurun_out/bench_$c.json | cut -c1-150
done
timeout 600 python bench.py --mode infer --no-cpu-baseline > gpurun_out/bench_C3R_infer.json 2> gpurun_out/bench_C3R.err
tail -1 gpurun_out/bench_C3R_infer.json | cut -c1-150
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>&1; tail -1 gpurun_out/bench_reference.json | cut -c1-150

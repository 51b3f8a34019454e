#!/bin/bash
# repeat the default bench N times; print value, ms/step, sum of phases, clocks
for i in $(seq ${N:-3}); do
timeout 200 python bench.py --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu-baseline $EXTRA 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']
print(round(d['value']), d['ms_per_step'], 'phases', round(sum(p.values()),2), {k: round(v,2) for k,v in p.items()}, d['clocks'])"
done

#!/bin/bash
# BVH build time per step over library variants: VS="tag ..." (C3 bench, 5 timed steps)
summ() {
python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']
print('$1', round(d['value']), d['ms_per_step'], 'build', p['build'], 'trace', p['trace'], 'visits', d['counters_per_step']['node_visits'])"
}
timeout 150 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ base
for v in $VS; do
  DT_LIBDIFFTRANS=paper_2603_00413_b200/variants/libdifftrans_$v.so timeout 150 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ $v
done

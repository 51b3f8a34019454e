#!/bin/bash
# C3 bench over library variants: VS="tag ..." (paper_2603_00413_b200/variants/libdifftrans_<tag>.so)
summ() {
python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']
print('$1', round(d['value']), d['ms_per_step'], 'trace0', p['trace0'], 'trace', p['trace'], 'shade', p['shade'], 'bwd', p['bwd'], 'gather', p['gather'], 'visits', d['counters_per_step']['node_visits'], 'tris', d['counters_per_step']['tri_tests'])"
}
timeout 150 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ base
for v in $VS; do
  DT_LIBDIFFTRANS=paper_2603_00413_b200/variants/libdifftrans_$v.so timeout 150 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ $v
done

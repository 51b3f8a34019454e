#!/bin/bash
# C3 bench over environment settings: ENVS="tag:VAR=x,VAR2=y ..." (one bench per entry)
summ() {
python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']; c=d['counters_per_step']
print('$1', round(d['value']), d['ms_per_step'], 'trace0', p['trace0'], 'trace', p['trace'], 'shade', p['shade'], 'bwd', p['bwd'], 'visits', c['node_visits'], 'tris', c['tri_tests'])"
}
CFG=${CFG:-C3}
for e in $ENVS; do
  tag=${e%%:*}; vars=${e#*:}
  env $(echo $vars | tr ',' ' ') timeout 150 python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ $tag
done

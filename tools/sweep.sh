#!/bin/bash
# traversal tuning sweep (C3 bench, no e2e/cpu baseline)
summ() {
python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']; c=d['counters_per_step']
print('$1', round(d['value']), d['ms_per_step'], 'trace0', p['trace0'], 'trace', p['trace'], 'shade', p['shade'], 'bwd', p['bwd'], 'visits', c['node_visits'], 'tris', c['tri_tests'])"
}
for lm in ${LEAVES:-1 2 3}; do for mode in ${MODES:-0 1 2}; do
  DT_LEAF_MAX=$lm DT_TRAV_MODE=$mode timeout 120 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ "leaf=$lm mode=$mode"
done; done
for ch in ${CHUNKS:-64 128 512 1024}; do
  DT_LEAF_MAX=${CLEAF:-2} DT_TRAV_MODE=2 DT_TRAV_CHUNK=$ch timeout 120 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ "chunk=$ch"
done

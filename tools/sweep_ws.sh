#!/bin/bash
# warp-synchronous traversal sweep
summ() {
python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']; c=d['counters_per_step']
print('$1', round(d['value']), d['ms_per_step'], 'trace0', p['trace0'], 'trace', p['trace'], 'visits', c['node_visits'], 'tris', c['tri_tests'])"
}
DT_TRAV_MODE=3 DT_LEAF_VOTE=16 timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "c1_full or c2_grid or sigma_grid or flat" --timeout 300 2>&1 | tail -1
for cfg in "1 1 32" "3 1 32" "3 1 24" "3 1 16" "3 2 32" "3 2 24" "3 3 24"; do
  set -- $cfg
  DT_TRAV_MODE=$1 DT_LEAF_MAX=$2 DT_LEAF_VOTE=$3 timeout 100 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ "mode=$1 leaf=$2 vote=$3"
done

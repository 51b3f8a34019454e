#!/bin/bash
# Variant sweep on the GPU box: tools/sweep.sh CONFIG tag1 tag2 ...  (variants built here with
# tools/build_variants.py tag=DEF1,DEF2 ...); prints value, ms/step and the phase split.
CFG=${1:-C3}; shift
summ() {
python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']; c=d['counters_per_step']
print('$1', round(d['value']), d['ms_per_step'], 'trace0', p['trace0'], 'trace', p['trace'], 'shade', p['shade'], 'bwd', p['bwd'], 'visits', c['node_visits'], 'tris', c['tri_tests'])"
}
export BENCH_NO_CLOCKS=1
timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ default
for v in "$@"; do
  timeout 300 python tools/bench_variant.py paper_2603_00413_b200/variants/libdifftrans_$v.so --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ "$v"
done

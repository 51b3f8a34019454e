#!/bin/bash
# sigma-walk group size sweep (C4 bench): default build (G=8) + variants
summ() {
python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']
print('$1', round(d['value']), d['ms_per_step'], 'shade', p['shade'], 'bwd', p['bwd'], 'trace', p['trace'])"
}
timeout 200 python bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ "default"
for g in ${GS:-b2 b8 f4 f16}; do
  DT_LIBDIFFTRANS=paper_2603_00413_b200/variants/libdifftrans_g$g.so timeout 200 python bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ "G=$g"
done

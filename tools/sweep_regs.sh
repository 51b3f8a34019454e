#!/bin/bash
# register-cap sweep of the sigma-grid kernel variants (C4 bench)
summ() {
python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']
print('$1', round(d['value'],1), d['ms_per_step'], 'shade', p['shade'], 'bwd', p['bwd'])"
}
timeout 200 python bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ "default"
for v in ${VS:-s80 s96 s112 s128 b96 b112}; do
  DT_LIBDIFFTRANS=paper_2603_00413_b200/variants/libdifftrans_$v.so timeout 200 python bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ "$v"
done

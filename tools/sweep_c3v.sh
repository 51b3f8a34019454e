#!/bin/bash
summ() {
python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']
print('$1', round(d['value']), d['ms_per_step'], 'trace0', p['trace0'], 'shade', p['shade'], 'bwd', p['bwd'])"
}
timeout 300 python bench.py --config C3V --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ base
for v in $VS; do
  DT_LIBDIFFTRANS=paper_2603_00413_b200/variants/libdifftrans_$v.so timeout 300 python bench.py --config C3V --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ $v
done

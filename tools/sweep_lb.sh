#!/bin/bash
# launch-bounds variants (tools: build with paper_2603_00413_b200/build.py defines/out)
summ() {
python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['phase_ms_per_step']
print('$1', round(d['value']), d['ms_per_step'], 'trace0', p['trace0'], 'trace', p['trace'], 'shade', p['shade'], 'bwd', p['bwd'], 'gather', p['gather'])"
}
timeout 150 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ base
for v in ${VARIANTS:-t10 t12 s8 s12 b6 b8}; do
  DT_LIBDIFFTRANS=paper_2603_00413_b200/variants/libdifftrans_$v.so timeout 150 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | summ $v
done

#!/bin/bash
# GPU box: rebuild libdifftrans.so in place with the in-kernel bounds checks (-DDT_CHECKED=1)
# and run the GPU test suite with DT_CHECKED_RUN=1 (conftest asserts after every test that no
# check failed), plus the sanitizer workload (tools/sanitize_run.py).  compute-sanitizer is
# closed on the GPU pool; this is its substitute for out-of-bounds indexing.
mkdir -p gpurun_out
# self-test of the plumbing: a build whose k_gather fails a check must report it
python -c "from paper_2603_00413_b200 import build as B; B.build(force=True, defines=['DT_CHECKED=1', 'DT_CHECK_SELFTEST=1'])" || exit 1
python -c "
import __graft_entry__ as g
from paper_2603_00413_b200 import _native as N
try:
    g.smoke()
except AssertionError:
    pass
st = N.check_status(); print('self-test (a failing check compiled into k_gather):', st); assert st['trace'] > 0
" || { echo "check self-test FAILED"; exit 1; }
python -c "from paper_2603_00413_b200 import build as B; B.build(force=True, defines=['DT_CHECKED=1'])" || exit 1
python -c "from paper_2603_00413_b200 import _native as N; print('check status (checked build):', N.check_status())"
DT_CHECKED_RUN=1 timeout ${PT:-2400} python -m pytest tests/ -q -m gpu -p no:cacheprovider ${PYARGS} > gpurun_out/checked_tests.log 2>&1
echo "checked pytest rc=$?"; tail -3 gpurun_out/checked_tests.log
python tools/sanitize_run.py > gpurun_out/checked_workload.log 2>&1
python -c "from paper_2603_00413_b200 import _native as N; print('check status after workload:', N.check_status())" >> gpurun_out/checked_workload.log 2>&1
tail -2 gpurun_out/checked_workload.log

#!/bin/bash
# GPU box: the four compute-sanitizer tools over tools/sanitize_run.py; logs in gpurun_out/
mkdir -p gpurun_out
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 50 --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|========= (Invalid|Race|Barrier)" gpurun_out/sanitize_$t.log | head -5
done

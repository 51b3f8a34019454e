#!/bin/bash
# GPU box: ncu source-counter captures of one C3 traversal launch for the in-tree library and
# each named variant (tools/build_variants.py): tools/ncu_variants.sh KERNEL_REGEX SKIP tag1 tag2 ...
K=${1:-k_traverse_level}; S=${2:-16}; shift 2
mkdir -p gpurun_out
B="--config ${CFG:-C3} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
SEC="--section SourceCounters --section LaunchStats --section Occupancy --section SchedulerStats --section WarpStateStats --section ComputeWorkloadAnalysis --section MemoryWorkloadAnalysis --section SpeedOfLight"
export BENCH_NO_CLOCKS=1
timeout 900 ncu $SEC --clock-control none --import-source on -k regex:$K -s $S -c 1 -f -o gpurun_out/${P:-nv}_default python bench.py $B > gpurun_out/${P:-nv}_default.log 2>&1
echo "default rc=$?"
for v in "$@"; do
  timeout 900 ncu $SEC --clock-control none --import-source on -k regex:$K -s $S -c 1 -f -o gpurun_out/${P:-nv}_$v python tools/bench_variant.py paper_2603_00413_b200/variants/libdifftrans_$v.so $B > gpurun_out/${P:-nv}_$v.log 2>&1
  echo "$v rc=$?"
done

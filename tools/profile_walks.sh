#!/bin/bash
# GPU box: ncu --set full of one texture-walk backward launch and one walk shade launch at C4
# (sigma grid) and C4H (hash texture), for the walks' L2 roofline (bench.py "bound": "l2").
# Scratch in gpurun_out/; tools/ncu_summary.py turns it into profiles/.  Usage: profile_walks.sh TAG
T=${1:-r02w}
export BENCH_NO_CLOCKS=1
for c in C4 C4H; do
  B="python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
  k=$([ $c = C4 ] && echo grid || echo hash)
  # skip the first warm-up step's 7 backward launches; capture a level-1 launch of the second
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_backward_level_$k -s 8 -c 1 \
    -o gpurun_out/${T}_${c}_bwd $B > gpurun_out/${T}_${c}_ncu_bwd.log 2>&1
  echo "$c bwd rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_shade_level_$k -s 8 -c 1 \
    -o gpurun_out/${T}_${c}_shade $B > gpurun_out/${T}_${c}_ncu_shade.log 2>&1
  echo "$c shade rc=$?"
  ncu -i gpurun_out/${T}_${c}_bwd.ncu-rep --page raw --csv 2>/dev/null | head -1 | tr ',' '\n' | grep -i "red\|atom" | head -40 > gpurun_out/${T}_${c}_red_metric_names.txt
done
# DRAM traffic of every backward launch of one step (the second warm-up step's 7 launches at
# D = 6) -> tools/ncu_traffic.py -> profiles/r02_traffic_<config>.json (the bench's "traffic")
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,smsp__thread_inst_executed_per_inst_executed.ratio,sm__inst_executed.avg.per_cycle_active,smsp__issue_active.avg.pct_of_peak_sustained_active
for c in C4 C4H; do
  B="python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
  k=$([ $c = C4 ] && echo grid || echo hash)
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_backward_level_$k -s 7 -c 7 \
    -o gpurun_out/${T}_${c}_bwd_traffic $B > gpurun_out/${T}_${c}_ncu_traffic.log 2>&1
  echo "$c traffic rc=$?"
done

#!/bin/bash
# Round-2 ncu evidence (one GPU): the launch list of one timed step and --set full on
# the first 14 launches of the step's main kernels (rounds 0-2), through the
# stream-ordered path (ncu cannot profile kernel nodes of graphs with conditional
# nodes; the kernels are the same).
OUT=${OUT:-gpurun_out}
B="python bench.py --ncu --steps 1 --warmup 3 --no-cpu-baseline --tdg-queries 0"
export LF_SEARCH_GRAPH=0
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --profile-from-start off --csv --log-file $OUT/launches_full.csv $B > /dev/null 2>&1
echo "launch list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"lb_tile|leaf_order|scan_pq|pq_q8_bound|filter_tc|plan_warp|pq_tail_e1" -c 14 \
  -o $OUT/prof_r2 $B > $OUT/ncu_r2.log 2>&1
echo "full set rc=$?"

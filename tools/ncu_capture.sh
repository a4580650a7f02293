#!/bin/bash
# ncu evidence for profiles/ (run under gpurun, ONE GPU).  Passes over the real
# bench workload (25M x 256, cap 10K, 1000 queries); the profiling range is the
# timed step only (bench.py --ncu -> cudaProfilerStart/Stop).
#  1) launch list: every kernel of the timed step with its device time
#     (cold-cache, serialised: compare shares, not absolutes);
#  2) DRAM bytes of every leaf-scan launch of the step (-> roofline.traffic);
#  3) --set full on selected scan launches, the filter kernel and the bounds/sort;
#  4) --set full on the training-data-generation kernel (tools/tdg_probe.py, 2M x 1K).
OUT=${OUT:-gpurun_out}
EXTRA=${EXTRA:-}
B="python bench.py --ncu --steps 1 --warmup 3 --no-cpu-baseline --tdg-queries 0 $EXTRA"
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $OUT/launches.csv $B > $OUT/ncu_launches_bench.json 2> $OUT/ncu_launches.log
echo "launch list rc=$?"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --profile-from-start off -k regex:"${SCAN_REGEX:-scan_q8_kernel|scan_pq_kernel|pq_q8_bound_kernel|pq_tail_kernel}" --csv --log-file $OUT/scan_dram.csv \
    $B > $OUT/ncu_dram_bench.json 2> $OUT/ncu_dram.log
echo "scan dram rc=$?"
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"${KREGEX:-scan_q8_kernel|scan_pq_kernel|pq_q8_bound_kernel|pq_tail_kernel|filter_tc_kernel|bounds_sort_kernel|plan_warp_kernel}" \
    --launch-skip ${KSKIP:-0} -c ${KCOUNT:-8} -o $OUT/prof_full $B > $OUT/ncu_full.log 2>&1
echo "full set rc=$?"
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:mindist_q8 -c 1 \
    -o $OUT/prof_tdg python tools/tdg_probe.py 2000000 1024 q8 > $OUT/ncu_tdg.log 2>&1
echo "tdg full rc=$?"
ls -la $OUT

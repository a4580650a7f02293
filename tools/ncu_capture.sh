#!/bin/bash
# ncu evidence for profiles/ (run under gpurun, ONE GPU).  Two passes over the
# real bench workload (25M x 256, cap 10K, 1000 queries); the profiling range is
# the timed steps only (bench.py --ncu -> cudaProfilerStart/Stop).
#  1) launch list: every kernel of the timed steps with its device time
#     (cold-cache, serialised: compare shares, not absolutes);
#  2) --set full on the filter kernel and the first leaf-scan rounds.
OUT=${OUT:-gpurun_out}
EXTRA=${EXTRA:-}
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $OUT/launches.csv python bench.py --ncu --steps 1 --warmup 3 --no-cpu-baseline $EXTRA \
    > $OUT/ncu_bench.json 2> $OUT/ncu_bench.log
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"${KREGEX:-scan_ea2_kernel|filter_tc_kernel}" -c ${KCOUNT:-5} -o $OUT/prof_full \
    python bench.py --ncu --steps 1 --warmup 3 --no-cpu-baseline $EXTRA > $OUT/ncu_full.log 2>&1
echo "full set rc=$?"
ls -la $OUT

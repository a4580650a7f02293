#!/bin/bash
# One gpurun pass: GPU tests, the default bench line, and the ncu launch list of one
# timed step.  Outputs under gpurun_out/ with the given tag.
TAG=${1:-check}
OUT=gpurun_out
if [ -z "$SKIP_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/gputest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/gputest_$TAG.log
fi
timeout 600 python bench.py ${BENCH_ARGS:-} > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
if [ -z "$SKIP_NCU" ]; then
  # ncu cannot profile kernel nodes of graphs with conditional nodes: the launch list
  # runs the same kernels through the stream-ordered path (LF_SEARCH_GRAPH=0)
  LF_SEARCH_GRAPH=0 timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $OUT/launches_$TAG.csv python bench.py --ncu --steps 1 --warmup 3 --no-cpu-baseline --tdg-queries 0 \
    > /dev/null 2>&1; echo "ncu rc=$?"
fi

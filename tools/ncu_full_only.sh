#!/bin/bash
# --set full on selected kernels of the timed steps only (see ncu_capture.sh)
OUT=${OUT:-gpurun_out}
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:"${KREGEX:-scan_ea2_kernel}" -c ${KCOUNT:-4} -o $OUT/${NAME:-prof_scan} \
    python bench.py --ncu --steps 1 --warmup 3 --no-cpu-baseline --tdg-queries 0 ${EXTRA:-} > $OUT/${NAME:-prof_scan}.log 2>&1
echo "full set rc=$?"

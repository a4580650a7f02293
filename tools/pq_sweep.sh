# Ring-geometry sweep of scan_pq_kernel (rows per slot, slots per warp, warps per SM):
# rebuilds with each setting and times the bench workload with tools/step_probe.py.
# Run under gpurun from the repo root; leaves the last setting in the source.
F=paper_2502_01836_b200/csrc/scan_pq.cu
run() {
  sed -i "s/^#define LF_PQW_STG .*/#define LF_PQW_STG $1/; s/^#define LF_PQW_NS .*/#define LF_PQW_NS $2/; s/^#define LF_PQW_WARPS32 .*/#define LF_PQW_WARPS32 $3/" $F
  python -m paper_2502_01836_b200._build > /dev/null 2>&1 || { echo build-fail $*; return; }
  python tools/step_probe.py "cfg_$1_$2_$3" > gpurun_out/sw_$1_$2_$3.log 2>&1; tail -1 gpurun_out/sw_$1_$2_$3.log
}
run 64 4 16
run 32 4 32
run 32 6 24
run 64 3 20
run 64 4 16

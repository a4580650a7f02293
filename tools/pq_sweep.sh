F=paper_2502_01836_b200/csrc/scan_pq.cu
run() { sed -i "s/^#define LF_PQW_STG .*/#define LF_PQW_STG $1/; s/^#define LF_PQW_NS .*/#define LF_PQW_NS $2/; s/^#define LF_PQW_WARPS32 .*/#define LF_PQW_WARPS32 $3/; s/^#define LF_PQ_PREFETCH .*/#define LF_PQ_PREFETCH $4/" $F; python -m paper_2502_01836_b200._build > /dev/null 2>&1 || { echo build-fail $*; return; }; python tools/step_probe.py "cfg_$1_$2_$3_$4" > gpurun_out/sw_$1_$2_$3_$4.log 2>&1; tail -1 gpurun_out/sw_$1_$2_$3_$4.log; }
run 64 4 16 0

run 32 4 32 0
run 32 6 24 0
run 64 3 20 0

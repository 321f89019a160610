#!/bin/bash
# Profile of the default YFCC-shaped 0.90 operating point (launch list + ncu full of the top kernels), then f2 sweep.
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
Y="--widths 2 --and-scan 2000 --modes greedy --targets 0.90"
NCU_COUNT=6 bash scripts/r02_prof.sh r02s 'k_scan_tc|k_and_filter|k_graph' $Y
tail -n 30 gpurun_out/r02s_sum.log
timeout 1500 python scripts/f2_sweep.py > gpurun_out/r02s_f2.json 2> gpurun_out/r02s_f2.log; echo "f2 rc=$?"; tail -n 12 gpurun_out/r02s_f2.log
rm -rf $VF_GRAPH_CACHE

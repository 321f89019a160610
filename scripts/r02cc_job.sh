#!/bin/bash
# Profile of the YFCC-shaped 0.99 operating point (itopk 192, w 2, f3 50000): launch list, ncu full of
# the scan and graph kernels, TC-scan role cycle breakdown
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
Y="--widths 2 --and-scan 50000 --modes greedy --targets 0.99"
NCU_COUNT=2 bash scripts/r02_prof.sh r02cc 'k_scan_tc|k_graph|k_and_filter' $Y
tail -n 40 gpurun_out/r02cc_sum.log | grep -E "^\| \`|##|Top stall"
VF_NVCC_EXTRA=-DVF_TC_PROF timeout 900 python scripts/tc_prof.py --config yfcc --itopk 192 --and-scan 50000 --reps 1 > gpurun_out/r02cc_tcprof.log 2>&1
python -c "from paper_2506_00812_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
grep "TCPROF blk 0" gpurun_out/r02cc_tcprof.log | tail -n 12
rm -rf $VF_GRAPH_CACHE
# overlap policy A/B at both operating points (graph CTAs per SM cap, graph-first) vs serial
S="VF_GRAPH_PER_SM=0 VF_GRAPH_PER_SM=2 VF_GRAPH_PER_SM=3 VF_GRAPH_PER_SM=4 VF_GRAPH_PER_SM=5 VF_GRAPH_FIRST=1"
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 $S > gpurun_out/r02cc_ov32.log 2>&1; grep step gpurun_out/r02cc_ov32.log
timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 $S > gpurun_out/r02cc_ov192.log 2>&1; grep step gpurun_out/r02cc_ov192.log
timeout 900 python scripts/ab_env.py --config sift --itopk 16 --w 2 $S > gpurun_out/r02cc_ovs16.log 2>&1; grep step gpurun_out/r02cc_ovs16.log
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config sift --itopk 16 --w 2 VF_GRAPH_PER_SM=0 > gpurun_out/r02cc_ovs16s.log 2>&1; grep step gpurun_out/r02cc_ovs16s.log
rm -rf $VF_GRAPH_CACHE

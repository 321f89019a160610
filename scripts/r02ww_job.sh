#!/bin/bash
# L2 fetch granularity hint (VF_L2_FETCH, cudaLimitMaxL2FetchGranularity): graph DRAM bytes and step times
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ww_build.log 2>&1 || exit 1
Y="--widths 2 --and-scan 1000 --modes greedy --targets 0.90 --no-paper-timing"
timeout 900 python bench.py --lat-calls 0 --no-cpu-baseline $Y > /dev/null 2>&1
for g in 0 32 64 128; do
  VF_L2_FETCH=$g timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_graph|k_scan_tc|k_and_filter" -c 3 --csv python bench.py --no-cpu-baseline --lat-calls 0 --steps 2 --warmup 3 $Y > gpurun_out/r02ww_ncu_$g.csv 2> gpurun_out/r02ww_ncu_$g.log
  echo "fetch $g"; grep -E "dram__bytes_read|gpu__time" gpurun_out/r02ww_ncu_$g.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-160 | head -6
  VF_L2_FETCH=$g VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 VF_KNOBS=11 > gpurun_out/r02ww_ab_$g.log 2>&1; grep step gpurun_out/r02ww_ab_$g.log
done
rm -rf $VF_GRAPH_CACHE

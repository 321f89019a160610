#!/bin/bash
# graph DRAM bytes with and without the exact-size row prefetch (VF_KNOBS 11 vs 13), ncu full of k_graph at the 0.90 point
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02vv_build.log 2>&1 || exit 1
Y="--widths 2 --and-scan 1000 --modes greedy --targets 0.90 --no-paper-timing"
timeout 900 python bench.py --lat-calls 0 --no-cpu-baseline $Y > /dev/null 2>&1
for kn in 11 13; do
  VF_KNOBS=$kn timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_graph -c 2 --csv python bench.py --no-cpu-baseline --lat-calls 0 --steps 2 --warmup 3 $Y > gpurun_out/r02vv_ncu_$kn.csv 2> gpurun_out/r02vv_ncu_$kn.log
  echo "knobs $kn"; grep -E "dram__bytes|gpu__time|hit_rate" gpurun_out/r02vv_ncu_$kn.csv | cut -c1-220 | tail -8
done
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 VF_KNOBS=11 VF_KNOBS=13 VF_KNOBS=11 VF_KNOBS=13 > gpurun_out/r02vv_ab.log 2>&1; grep step gpurun_out/r02vv_ab.log
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 VF_KNOBS=11 VF_KNOBS=13 > gpurun_out/r02vv_ab192.log 2>&1; grep step gpurun_out/r02vv_ab192.log
rm -rf $VF_GRAPH_CACHE

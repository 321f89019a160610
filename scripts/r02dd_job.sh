#!/bin/bash
# overlap order A/B: graph from the fork (0) vs after the AND pre-filter (VF_GRAPH_AFTER=1) vs serial
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02dd_build.log 2>&1 || { tail -20 gpurun_out/r02dd_build.log; exit 1; }
S="VF_GRAPH_AFTER=0 VF_GRAPH_AFTER=1"
timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 $S > gpurun_out/r02dd_ov32.log 2>&1; grep step gpurun_out/r02dd_ov32.log
timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 $S > gpurun_out/r02dd_ov192.log 2>&1; grep step gpurun_out/r02dd_ov192.log
timeout 900 python scripts/ab_env.py --config yfcc --itopk 96 --w 2 --and-scan 10000 $S > gpurun_out/r02dd_ov96.log 2>&1; grep step gpurun_out/r02dd_ov96.log
timeout 900 python scripts/ab_env.py --config sift --itopk 16 --w 2 $S > gpurun_out/r02dd_ovs16.log 2>&1; grep step gpurun_out/r02dd_ovs16.log
timeout 900 python scripts/ab_env.py --config sift --itopk 48 --w 2 $S > gpurun_out/r02dd_ovs48.log 2>&1; grep step gpurun_out/r02dd_ovs48.log
rm -rf $VF_GRAPH_CACHE

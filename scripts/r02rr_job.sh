#!/bin/bash
# per-warp shared-memory budget of the graph kernel (VF_GRAPH_WARP_KB: visited-table slots vs resident CTAs)
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02rr_build.log 2>&1 || { tail -20 gpurun_out/r02rr_build.log; exit 1; }
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 VF_GRAPH_WARP_KB=7 VF_GRAPH_WARP_KB=8 VF_GRAPH_WARP_KB=9 VF_GRAPH_WARP_KB=10 VF_GRAPH_WARP_KB=12 VF_GRAPH_WARP_KB=14 > gpurun_out/r02rr_a.log 2>&1; grep step gpurun_out/r02rr_a.log
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 VF_GRAPH_WARP_KB=6 VF_GRAPH_WARP_KB=7 VF_GRAPH_WARP_KB=8 VF_GRAPH_WARP_KB=9 > gpurun_out/r02rr_b.log 2>&1; grep step gpurun_out/r02rr_b.log
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config sift --itopk 48 --w 2 VF_GRAPH_WARP_KB=6 VF_GRAPH_WARP_KB=7 VF_GRAPH_WARP_KB=8 VF_GRAPH_WARP_KB=9 > gpurun_out/r02rr_c.log 2>&1; grep step gpurun_out/r02rr_c.log
rm -rf $VF_GRAPH_CACHE

#!/bin/bash
# A/B of VF_KNOBS (filter signature loads, graph prefetch modes) on the YFCC-shaped operating points
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02t_build.log 2>&1 || { tail -20 gpurun_out/r02t_build.log; exit 1; }
K="VF_KNOBS=0 VF_KNOBS=1 VF_KNOBS=3 VF_KNOBS=5 VF_KNOBS=9 VF_KNOBS=11 VF_KNOBS=13"
timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 2000 $K > gpurun_out/r02t_ab32.log 2>&1; grep step gpurun_out/r02t_ab32.log
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 2000 $K > gpurun_out/r02t_ab32s.log 2>&1; grep step gpurun_out/r02t_ab32s.log
timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 VF_KNOBS=0 VF_KNOBS=1 VF_KNOBS=3 VF_KNOBS=11 > gpurun_out/r02t_ab192.log 2>&1; grep step gpurun_out/r02t_ab192.log
rm -rf $VF_GRAPH_CACHE

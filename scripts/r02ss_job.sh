#!/bin/bash
# overlap vs serial across f3 thresholds (VF_OVERLAP read per search; default 2 = serial from f3 >= 20000)
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ss_build.log 2>&1 || { tail -20 gpurun_out/r02ss_build.log; exit 1; }
S="VF_OVERLAP=1 VF_OVERLAP=0"
for cfg in "32 2 1000" "28 2 2000" "64 2 5000" "112 2 10000" "192 2 20000" "192 2 50000" "448 4 20000"; do
  set -- $cfg
  timeout 900 python scripts/ab_env.py --config yfcc --itopk $1 --w $2 --and-scan $3 $S > gpurun_out/r02ss_$1_$3.log 2>&1; echo "itopk $1 w $2 f3 $3"; grep step gpurun_out/r02ss_$1_$3.log
done
rm -rf $VF_GRAPH_CACHE

#!/bin/bash
# 128-B K chunks for the TC scan (VF_TC_CW=128): parity of the scan tests under it + A/B vs the default
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ee_build.log 2>&1 || { tail -20 gpurun_out/r02ee_build.log; exit 1; }
VF_TC_CW=128 timeout 900 python -m pytest tests/test_gpu_scan_tc.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r02ee_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02ee_pytest.log; tail -n 4 gpurun_out/r02ee_pytest.log
for cw in 0 128; do
  echo "== VF_TC_CW=$cw"
  VF_TC_CW=$cw VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 VF_KNOBS=11 > gpurun_out/r02ee_y32s_$cw.log 2>&1; grep step gpurun_out/r02ee_y32s_$cw.log
  VF_TC_CW=$cw VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 VF_KNOBS=11 > gpurun_out/r02ee_y192s_$cw.log 2>&1; grep step gpurun_out/r02ee_y192s_$cw.log
done
rm -rf $VF_GRAPH_CACHE

#!/bin/bash
# parity + A/B of the grouped segment collapse (k_collect)
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02w_build.log 2>&1 || { tail -20 gpurun_out/r02w_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scan_tc.py -m gpu -x -q > gpurun_out/r02w_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02w_pytest.log; tail -n 4 gpurun_out/r02w_pytest.log
K="VF_COLLAPSE=0 VF_COLLAPSE=1"
timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 2000 $K > gpurun_out/r02w_ab32.log 2>&1; grep step gpurun_out/r02w_ab32.log
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 2000 $K > gpurun_out/r02w_ab32s.log 2>&1; grep step gpurun_out/r02w_ab32s.log
timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 $K > gpurun_out/r02w_ab192.log 2>&1; grep step gpurun_out/r02w_ab192.log
timeout 900 python scripts/ab_env.py --config yfcc --itopk 96 --w 2 --and-scan 10000 $K > gpurun_out/r02w_ab96.log 2>&1; grep step gpurun_out/r02w_ab96.log
rm -rf $VF_GRAPH_CACHE

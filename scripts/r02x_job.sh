#!/bin/bash
# A/B: f3 pre-filter tile size x segment regrouping; parity subset
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02x_build.log 2>&1 || { tail -20 gpurun_out/r02x_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scan_tc.py -m gpu -x -q > gpurun_out/r02x_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02x_pytest.log; tail -n 4 gpurun_out/r02x_pytest.log
K="VF_F3_TILE=2048,VF_COLLAPSE=0 VF_F3_TILE=2048,VF_COLLAPSE=1 VF_F3_TILE=4096,VF_COLLAPSE=0 VF_F3_TILE=8192,VF_COLLAPSE=0 VF_F3_TILE=16384,VF_COLLAPSE=0 VF_F3_TILE=8192,VF_COLLAPSE=1"
timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 2000 $K > gpurun_out/r02x_ab32.log 2>&1; grep step gpurun_out/r02x_ab32.log
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 2000 $K > gpurun_out/r02x_ab32s.log 2>&1; grep step gpurun_out/r02x_ab32s.log
timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 $K > gpurun_out/r02x_ab192.log 2>&1; grep step gpurun_out/r02x_ab192.log
rm -rf $VF_GRAPH_CACHE

#!/bin/bash
# parity of the AND pre-filter rewrite (filter tile list, parallel label setup) + A/B (occupancy knob)
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02u_build.log 2>&1 || { tail -20 gpurun_out/r02u_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scan_tc.py -m gpu -x -q > gpurun_out/r02u_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02u_pytest.log; tail -n 4 gpurun_out/r02u_pytest.log
K="VF_KNOBS=11 VF_KNOBS=27 VF_KNOBS=10"
timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 2000 $K > gpurun_out/r02u_ab32.log 2>&1; grep step gpurun_out/r02u_ab32.log
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 2000 $K > gpurun_out/r02u_ab32s.log 2>&1; grep step gpurun_out/r02u_ab32s.log
timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 $K > gpurun_out/r02u_ab192.log 2>&1; grep step gpurun_out/r02u_ab192.log
rm -rf $VF_GRAPH_CACHE

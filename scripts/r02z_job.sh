#!/bin/bash
# A/B: bitmap-span path of the AND pre-filter (VF_KNOBS bit 5) and signature loads (bit 0); parity subset
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02z_build.log 2>&1 || { tail -20 gpurun_out/r02z_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scan_tc.py -m gpu -x -q > gpurun_out/r02z_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02z_pytest.log; tail -n 4 gpurun_out/r02z_pytest.log
K="VF_KNOBS=43 VF_KNOBS=11 VF_KNOBS=42 VF_KNOBS=10"
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 $K > gpurun_out/r02z_ab32s.log 2>&1; grep step gpurun_out/r02z_ab32s.log
timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 $K > gpurun_out/r02z_ab32.log 2>&1; grep step gpurun_out/r02z_ab32.log
timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 $K > gpurun_out/r02z_ab192.log 2>&1; grep step gpurun_out/r02z_ab192.log
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 $K > gpurun_out/r02z_ab192s.log 2>&1; grep step gpurun_out/r02z_ab192s.log
for mb in 6 7; do VF_LIB=abl/lib_minb$mb.so timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 VF_KNOBS=11 > gpurun_out/r02z_minb$mb.log 2>&1; echo "minb$mb"; grep step gpurun_out/r02z_minb$mb.log; done
rm -rf $VF_GRAPH_CACHE

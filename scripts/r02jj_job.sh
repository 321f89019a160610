#!/bin/bash
# next-parent adjacency prefetch (VF_KNOBS bit 5) A/B + the knob-equivalence parity test
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02jj_build.log 2>&1 || { tail -20 gpurun_out/r02jj_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "switches or overflow" > gpurun_out/r02jj_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02jj_pytest.log; tail -n 3 gpurun_out/r02jj_pytest.log
K="VF_KNOBS=11 VF_KNOBS=43"
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 $K > gpurun_out/r02jj_a.log 2>&1; grep step gpurun_out/r02jj_a.log
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 $K > gpurun_out/r02jj_b.log 2>&1; grep step gpurun_out/r02jj_b.log
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config sift --itopk 16 --w 2 $K > gpurun_out/r02jj_c.log 2>&1; grep step gpurun_out/r02jj_c.log
VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config sift --itopk 48 --w 2 $K > gpurun_out/r02jj_d.log 2>&1; grep step gpurun_out/r02jj_d.log
rm -rf $VF_GRAPH_CACHE

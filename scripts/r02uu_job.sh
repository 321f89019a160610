#!/bin/bash
# 3-chunk graph kernel instance for 192-B rows (VF_GRAPH_CPL3=0: the 4-chunk one): parity + A/B
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02uu_build.log 2>&1 || { tail -20 gpurun_out/r02uu_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_small.py tests/test_gpu_graph_build.py -m gpu -x -q > gpurun_out/r02uu_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02uu_pytest.log; tail -n 3 gpurun_out/r02uu_pytest.log
for v in 1 0; do
  echo "== VF_GRAPH_CPL3=$v"
  VF_GRAPH_CPL3=$v VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 VF_KNOBS=11 > gpurun_out/r02uu_a_$v.log 2>&1; grep step gpurun_out/r02uu_a_$v.log
  VF_GRAPH_CPL3=$v VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 VF_KNOBS=11 > gpurun_out/r02uu_b_$v.log 2>&1; grep step gpurun_out/r02uu_b_$v.log
done
rm -rf $VF_GRAPH_CACHE

#!/bin/bash
# TC scan pipeline depth: layout for 1 CTA per SM (qg 32, 5 stages) vs 2 CTAs (qg 16, 2 stages), 64-B vs 128-B chunks
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ff_build.log 2>&1 || { tail -20 gpurun_out/r02ff_build.log; exit 1; }
VF_TC_LAYOUT_CTAS=1 timeout 900 python -m pytest tests/test_gpu_scan_tc.py -m gpu -x -q > gpurun_out/r02ff_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02ff_pytest.log; tail -n 3 gpurun_out/r02ff_pytest.log
for v in "VF_TC_LAYOUT_CTAS=2" "VF_TC_LAYOUT_CTAS=1" "VF_TC_LAYOUT_CTAS=1 VF_TC_CW=128"; do
  echo "== $v"
  env $v VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 VF_KNOBS=11 > gpurun_out/r02ff_a.log 2>&1; grep step gpurun_out/r02ff_a.log
  env $v VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 VF_KNOBS=11 > gpurun_out/r02ff_b.log 2>&1; grep step gpurun_out/r02ff_b.log
  env $v timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 VF_KNOBS=11 > gpurun_out/r02ff_c.log 2>&1; grep step gpurun_out/r02ff_c.log
  env $v timeout 900 python scripts/ab_env.py --config sift --itopk 16 --w 2 VF_KNOBS=11 > gpurun_out/r02ff_d.log 2>&1; grep step gpurun_out/r02ff_d.log
done
rm -rf $VF_GRAPH_CACHE

#!/bin/bash
# beam search AND predicate resolved per item (bitmap pointers, signature mask) + direct-bitmap switch (VF_KNOBS bit 8)
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02mm_build.log 2>&1 || { tail -20 gpurun_out/r02mm_build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_small.py -m gpu -x -q > gpurun_out/r02mm_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02mm_pytest.log; tail -n 3 gpurun_out/r02mm_pytest.log
for lib in default abl/lib_head3.so; do
  if [ "$lib" = default ]; then unset VF_LIB; else export VF_LIB=$lib; fi
  echo "== $lib"
  VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 VF_KNOBS=11 VF_KNOBS=267 > gpurun_out/r02mm_a_$(basename $lib).log 2>&1; grep step gpurun_out/r02mm_a_$(basename $lib).log
  VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 0 VF_KNOBS=11 VF_KNOBS=267 > gpurun_out/r02mm_b_$(basename $lib).log 2>&1; grep step gpurun_out/r02mm_b_$(basename $lib).log
  VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 VF_KNOBS=11 VF_KNOBS=267 > gpurun_out/r02mm_c_$(basename $lib).log 2>&1; grep step gpurun_out/r02mm_c_$(basename $lib).log
done
unset VF_LIB
rm -rf $VF_GRAPH_CACHE

#!/bin/bash
# AND pre-filter: 6 rows per thread per round (abl/lib_filt6.so) vs 4; parity of the scan tests under the variant
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02zz_build.log 2>&1 || exit 1
VF_LIB=abl/lib_filt6.so timeout 900 python -m pytest tests/test_gpu_scan_tc.py -m gpu -x -q > gpurun_out/r02zz_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02zz_pytest.log; tail -n 2 gpurun_out/r02zz_pytest.log
for lib in default abl/lib_filt6.so; do
  if [ "$lib" = default ]; then unset VF_LIB; else export VF_LIB=$lib; fi
  echo "== $lib"
  VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 VF_KNOBS=11 VF_KNOBS=11 > gpurun_out/r02zz_a_$(basename $lib).log 2>&1; grep step gpurun_out/r02zz_a_$(basename $lib).log
  VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 VF_KNOBS=11 > gpurun_out/r02zz_b_$(basename $lib).log 2>&1; grep step gpurun_out/r02zz_b_$(basename $lib).log
done
unset VF_LIB
rm -rf $VF_GRAPH_CACHE

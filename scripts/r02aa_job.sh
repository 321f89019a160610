#!/bin/bash
# parity of the single-pass visited insert + A/B (VF_KNOBS bit 6) x graph register budget (VF_GRAPH_MINB 8/7/6)
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02aa_build.log 2>&1 || { tail -20 gpurun_out/r02aa_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_small.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/r02aa_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02aa_pytest.log; tail -n 4 gpurun_out/r02aa_pytest.log
for lib in default abl/lib_minb7.so abl/lib_minb6.so; do
  if [ "$lib" = default ]; then unset VF_LIB; else export VF_LIB=$lib; fi
  echo "== $lib"
  VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 1000 VF_KNOBS=11 VF_KNOBS=75 > gpurun_out/r02aa_y32_$(basename $lib).log 2>&1; grep step gpurun_out/r02aa_y32_$(basename $lib).log
  VF_OVERLAP=0 timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 VF_KNOBS=11 VF_KNOBS=75 > gpurun_out/r02aa_y192_$(basename $lib).log 2>&1; grep step gpurun_out/r02aa_y192_$(basename $lib).log
  timeout 900 python scripts/ab_env.py --config sift --itopk 16 --w 2 VF_KNOBS=11 VF_KNOBS=75 > gpurun_out/r02aa_s16_$(basename $lib).log 2>&1; grep step gpurun_out/r02aa_s16_$(basename $lib).log
  timeout 900 python scripts/ab_env.py --config sift --itopk 48 --w 2 VF_KNOBS=11 VF_KNOBS=75 > gpurun_out/r02aa_s48_$(basename $lib).log 2>&1; grep step gpurun_out/r02aa_s48_$(basename $lib).log
done
unset VF_LIB
rm -rf $VF_GRAPH_CACHE

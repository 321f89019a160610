#!/bin/bash
# final build: generic fp32 kernels on SIFT-like (FFMA scan, fp32 graph rows) and the f2 T sweep
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02xx_build.log 2>&1 || exit 1
VF_U8_STORE=0 VF_SCAN_TC=0 timeout 900 python bench.py --config sift --lat-calls 0 --no-cpu-baseline > gpurun_out/r02xx_bench_sift_fp32.json 2> gpurun_out/r02xx_bench_sift_fp32.log; echo "fp32 rc=$?"; tail -n 1 gpurun_out/r02xx_bench_sift_fp32.log
timeout 1800 python scripts/f2_sweep.py > gpurun_out/r02xx_f2.json 2> gpurun_out/r02xx_f2.log; echo "f2 rc=$?"; grep -v itopk gpurun_out/r02xx_f2.log | tail -n 16

#!/bin/bash
# Round-2 validation: whole GPU suite, default bench (YFCC-shaped), profile, SIFT-like + generic fp32
# benches, compute-sanitizer on tiny inputs
set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02y_build.log 2>&1 || { tail -20 gpurun_out/r02y_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02y_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02y_pytest.log; tail -n 3 gpurun_out/r02y_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02y_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02y_smoke.log; tail -n 2 gpurun_out/r02y_smoke.log
timeout 1200 python bench.py > gpurun_out/r02y_bench_yfcc.json 2> gpurun_out/r02y_bench_yfcc.log; echo "bench rc=$?" >> gpurun_out/r02y_bench_yfcc.log; tail -n 1 gpurun_out/r02y_bench_yfcc.log
Y="--widths 2 --and-scan 2000 --modes greedy --targets 0.90"
NCU_COUNT=3 bash scripts/r02_prof.sh r02y 'k_scan_tc|k_and_filter|k_graph' $Y
tail -n 12 gpurun_out/r02y_sum.log
timeout 900 python bench.py --config sift > gpurun_out/r02y_bench_sift.json 2> gpurun_out/r02y_bench_sift.log; echo "sift rc=$?" >> gpurun_out/r02y_bench_sift.log; tail -n 1 gpurun_out/r02y_bench_sift.log
VF_U8_STORE=0 VF_SCAN_TC=0 timeout 900 python bench.py --config sift --lat-calls 0 --no-cpu-baseline > gpurun_out/r02y_bench_sift_fp32.json 2> gpurun_out/r02y_bench_sift_fp32.log; echo "fp32 rc=$?" >> gpurun_out/r02y_bench_sift_fp32.log; tail -n 1 gpurun_out/r02y_bench_sift_fp32.log
bash scripts/r02_sanitize.sh r02y
rm -rf $VF_GRAPH_CACHE

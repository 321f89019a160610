#!/bin/bash
# Final round-2 measurement: the driver's commands (GPU tests, smoke, default bench, reference arm), then a
# launch list + ncu full of the default 0.90 point and the SIFT-like bench
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02tt_build.log 2>&1 || { tail -20 gpurun_out/r02tt_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02tt_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02tt_pytest.log; tail -n 3 gpurun_out/r02tt_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02tt_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02tt_smoke.log; tail -n 2 gpurun_out/r02tt_smoke.log
export VF_GRAPH_CACHE=/tmp/vf_graph_cache_$$
s=$(date +%s); timeout 1200 python bench.py > gpurun_out/r02tt_bench_yfcc.json 2> gpurun_out/r02tt_bench_yfcc.log; echo "bench rc=$? s=$(( $(date +%s) - s ))" >> gpurun_out/r02tt_bench_yfcc.log; tail -n 1 gpurun_out/r02tt_bench_yfcc.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02tt_ref.json 2> gpurun_out/r02tt_ref.log; echo "ref rc=$?" >> gpurun_out/r02tt_ref.log
OP=$(python -c "import json; j=json.load(open('gpurun_out/r02tt_bench_yfcc.json')); c=j['config']; print(f\"--widths {c['search_width']} --and-scan {c['and_scan_threshold']} --modes {c['recall_mode']} --targets 0.90\")")
echo "op: $OP"
NCU_COUNT=3 bash scripts/r02_prof.sh r02tt 'k_scan_tc|k_and_filter|k_graph' $OP
timeout 900 python bench.py --config sift > gpurun_out/r02tt_bench_sift.json 2> gpurun_out/r02tt_bench_sift.log; echo "sift rc=$?" >> gpurun_out/r02tt_bench_sift.log
NCU_COUNT=2 bash scripts/r02_prof.sh r02tt_sift 'k_graph|k_scan_tc' --config sift --widths 2 --targets 0.90
rm -rf $VF_GRAPH_CACHE

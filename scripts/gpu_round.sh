#!/bin/bash
# One gpurun job: SIFT-like bench + ncu launch list + full captures, then the same for YFCC-shaped.
# usage: scripts/gpu_round.sh TAG [sift|yfcc|both]
set -u
tag=$1; which=${2:-both}
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache
if [ "$which" != yfcc ]; then
  timeout 600 python bench.py > gpurun_out/${tag}_bench_sift.json 2> gpurun_out/${tag}_bench_sift.log
  timeout 600 scripts/profile.sh launches ${tag}_sift --widths 2 --steps 3 --warmup 3
  NCU_COUNT=4 timeout 900 scripts/profile.sh full ${tag}_sift 'k_graph|k_scan_tc' --widths 2 --steps 2 --warmup 3
fi
if [ "$which" != sift ]; then
  Y="--config yfcc --widths 2 --and-scan 2000 --gt-sample 2000"
  timeout 1500 python bench.py --config yfcc > gpurun_out/${tag}_bench_yfcc.json 2> gpurun_out/${tag}_bench_yfcc.log
  timeout 900 scripts/profile.sh launches ${tag}_yfcc $Y --steps 2 --warmup 3
  NCU_COUNT=6 timeout 1500 scripts/profile.sh full ${tag}_yfcc 'k_graph|k_scan_tc|k_hs_filter' $Y --steps 2 --warmup 3
fi

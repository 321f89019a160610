#!/bin/bash
# YFCC-shaped A/B of an env knob at the 0.90 operating point (graphs built once per job):
#   scripts/yfcc_ab.sh TAG "ENV=A" "ENV=B"
tag=$1; shift
export VF_GRAPH_CACHE=/tmp/vfc
A="--config yfcc --widths 2 --and-scan 2000 --gt-sample 2000 --lat-calls 0 --no-cpu-baseline --steps 10"
i=0
for e in "$@"; do
  env $e timeout 1200 python bench.py $A > gpurun_out/${tag}_$i.json 2> gpurun_out/${tag}_$i.log
  i=$((i+1))
done

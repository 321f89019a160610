#!/bin/bash
# A/B of the scan/graph overlap knobs on the SIFT-like bench (writes gpurun_out/ab_*.json)
# fields: VF_OVERLAP VF_TC_CTAS VF_GRAPH_FIRST VF_GRAPH_PER_SM
A="--widths 2 --lat-calls 0 --no-cpu-baseline --steps 20 $*"
for cfg in "0 2 0 0" "1 2 0 0" "1 1 1 4" "1 1 1 5" "1 2 1 1" "1 1 1 3"; do
  set -- $cfg
  VF_OVERLAP=$1 VF_TC_CTAS=$2 VF_GRAPH_FIRST=$3 VF_GRAPH_PER_SM=$4 timeout 300 python bench.py $A \
    > gpurun_out/ab_$1_$2_$3_$4.json 2> gpurun_out/ab_$1_$2_$3_$4.log
done

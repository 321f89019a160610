#!/bin/bash
# A/B of two builds of libvecflow on the same bench: scripts/ab_lib.sh OTHER.so TAG [bench args]
other=$1; tag=$2; shift 2
A="--widths 2 --lat-calls 0 --no-cpu-baseline --steps 20 $*"
for r in 1 2; do
  timeout 300 python bench.py $A > gpurun_out/ab_${tag}_base$r.json 2> /dev/null
  VF_LIB=$other timeout 300 python bench.py $A > gpurun_out/ab_${tag}_other$r.json 2> /dev/null
done

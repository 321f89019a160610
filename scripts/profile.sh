#!/bin/bash
# Profiling recipe (run under gpurun, one GPU). Writes into gpurun_out/.
#   scripts/profile.sh launches [bench args...]   -> per-launch device times of our kernels
#   scripts/profile.sh full <kernel-regex> [bench args...] -> ncu --set full capture of that kernel
set -u
mode=$1; shift
mkdir -p gpurun_out
case $mode in
  launches)
    ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' --csv \
        --log-file gpurun_out/launches.csv python bench.py --no-cpu-baseline "$@" > gpurun_out/launches_bench.log 2>&1
    ;;
  full)
    kern=$1; shift
    ncu --set full --clock-control none --import-source on -k regex:"$kern" -s ${NCU_SKIP:-12} -c ${NCU_COUNT:-2} \
        -o gpurun_out/prof_${kern//[^a-z_]/} python bench.py --no-cpu-baseline "$@" > gpurun_out/prof_${kern//[^a-z_]/}.log 2>&1
    ;;
esac

#!/bin/bash
# Profiling recipe (run under gpurun, one GPU). Writes into gpurun_out/.
#   scripts/profile.sh launches TAG [bench args...]  -> per-launch device times of every kernel in the
#                                                      bench's timed steps (NVTX range "timed")
#   scripts/profile.sh full TAG <kernel-regex> [bench args...] -> ncu --set full capture of that
#                                                      kernel's launches inside the timed steps
set -u
mode=$1; tag=$2; shift 2
mkdir -p gpurun_out
case $mode in
  launches)
    ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/${tag}_launches.csv python bench.py --no-cpu-baseline --lat-calls 0 "$@" \
        > gpurun_out/${tag}_launches.log 2>&1
    ;;
  full)
    kern=$1; shift
    ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:"$kern" \
        -c ${NCU_COUNT:-2} -o gpurun_out/${tag}_full python bench.py --no-cpu-baseline --lat-calls 0 "$@" \
        > gpurun_out/${tag}_full.log 2>&1
    ;;
esac

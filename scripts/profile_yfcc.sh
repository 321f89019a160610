#!/bin/bash
# YFCC-shaped ncu captures in one process (graphs are built once): the launch list of a short bench
# run, then full captures of the scan, pre-filter and graph kernels at the 0.90 operating point.
# Run under gpurun; writes gpurun_out/yfcc_*.
set -u
mkdir -p gpurun_out
ARGS="--config yfcc --widths 2 --and-scan 2000 --steps 2 --warmup 3 --lat-calls 0 --no-cpu-baseline --gt-sample 2000"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'^k_' --csv \
    --log-file gpurun_out/yfcc_launches.csv python bench.py $ARGS > gpurun_out/yfcc_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k_scan_tc|k_hs_filter|k_graph<0' \
    -s ${NCU_SKIP:-60} -c ${NCU_COUNT:-4} -o gpurun_out/yfcc_full python bench.py $ARGS > gpurun_out/yfcc_full.log 2>&1

#!/bin/bash
# usage: scripts/r02_prof.sh TAG KERNEL_REGEX [bench args...]: launch list + ncu --set full of the timed steps
set -u
tag=$1; kern=$2; shift 2
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1
# warm the graph cache (and time the plain bench at the same operating point)
timeout 1200 python bench.py --lat-calls 0 --no-cpu-baseline --no-paper-timing "$@" > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.log
timeout 900 scripts/profile.sh launches ${tag} --no-paper-timing --steps 2 --warmup 3 "$@"
NCU_COUNT=${NCU_COUNT:-3} timeout 1500 scripts/profile.sh full ${tag} "$kern" --no-paper-timing --steps 2 --warmup 3 "$@"
python scripts/summarize_profile.py gpurun_out/${tag}_ncu.md --launches gpurun_out/${tag}_launches.csv --full gpurun_out/${tag}_full.ncu-rep > gpurun_out/${tag}_sum.log 2>&1
for k in k_scan_tc k_graph k_and_filter; do
  ncu -i gpurun_out/${tag}_full.ncu-rep --page source --csv -k regex:$k > gpurun_out/${tag}_src_${k}.csv 2>/dev/null
done
ls -la gpurun_out | grep $tag

#!/bin/bash
# usage: scripts/r02_job.sh TAG "pytest args or SKIP" "bench args;bench args;..."
set -u
tag=$1; pt=$2; benches=$3
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo "build failed"; tail -30 gpurun_out/${tag}_build.log; exit 1; }
if [ "$pt" != "SKIP" ]; then
  timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scan_tc.py tests/test_gpu_small.py tests/test_gpu_fullsize.py -m gpu -x -q $pt > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
  tail -n 5 gpurun_out/${tag}_pytest.log
fi
i=0
IFS=';' read -ra BS <<< "$benches"
for b in "${BS[@]}"; do
  [ -z "$b" ] && continue
  timeout 1800 python bench.py $b > gpurun_out/${tag}_bench$i.json 2> gpurun_out/${tag}_bench$i.log; echo "bench$i rc=$? args=$b" >> gpurun_out/${tag}_bench$i.log
  tail -n 2 gpurun_out/${tag}_bench$i.log
  i=$((i+1))
done

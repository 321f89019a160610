#!/bin/bash
# usage: scripts/r02_job2.sh TAG "bench args;bench args;..."  -- builder tests first, then all GPU tests, then benches
set -u
tag=$1; benches=$2
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo "build failed"; tail -30 gpurun_out/${tag}_build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_graph_build.py -x -q > gpurun_out/${tag}_pytest_gb.log 2>&1; echo "pytest_gb rc=$?" >> gpurun_out/${tag}_pytest_gb.log
tail -n 15 gpurun_out/${tag}_pytest_gb.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scan_tc.py tests/test_gpu_small.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
tail -n 5 gpurun_out/${tag}_pytest.log
i=0
IFS=';' read -ra BS <<< "$benches"
for b in "${BS[@]}"; do
  [ -z "$b" ] && continue
  timeout 1800 python bench.py $b > gpurun_out/${tag}_bench$i.json 2> gpurun_out/${tag}_bench$i.log; echo "bench$i rc=$? args=$b" >> gpurun_out/${tag}_bench$i.log
  grep -v "^\[bench\] greedy\|^\[bench\] parallel" gpurun_out/${tag}_bench$i.log | tail -n 6 | cut -c1-400
  i=$((i+1))
done

#!/bin/bash
# Round-2 GPU check: build, GPU tests, smoke, default bench (YFCC-shaped). usage: scripts/r02_check.sh TAG [pytest-args]
set -u
tag=$1; shift
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q "$@" > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 1800 python bench.py > gpurun_out/${tag}_bench_yfcc.json 2> gpurun_out/${tag}_bench_yfcc.log; echo "bench rc=$?" >> gpurun_out/${tag}_bench_yfcc.log
tail -3 gpurun_out/${tag}_pytest.log gpurun_out/${tag}_smoke.log gpurun_out/${tag}_bench_yfcc.log

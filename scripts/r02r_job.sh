#!/bin/bash
# Round-2 re-entry check: build, the whole GPU suite, smoke, the default bench (timed), the reference arm.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02r_build.log 2>&1 || { echo "build failed"; tail -30 gpurun_out/r02r_build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02r_smi.log
lscpu > gpurun_out/r02r_lscpu.log
s=$(date +%s)
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02r_pytest.log 2>&1; echo "pytest rc=$? s=$(( $(date +%s) - s ))" >> gpurun_out/r02r_pytest.log
tail -n 3 gpurun_out/r02r_pytest.log
s=$(date +%s)
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02r_smoke.log 2>&1; echo "smoke rc=$? s=$(( $(date +%s) - s ))" >> gpurun_out/r02r_smoke.log
tail -n 2 gpurun_out/r02r_smoke.log
s=$(date +%s)
timeout 2400 python bench.py > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.log; echo "bench rc=$? s=$(( $(date +%s) - s ))" >> gpurun_out/r02r_bench.log
tail -n 2 gpurun_out/r02r_bench.log
s=$(date +%s)
timeout 1200 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02r_ref.json 2> gpurun_out/r02r_ref.log; echo "ref rc=$? s=$(( $(date +%s) - s ))" >> gpurun_out/r02r_ref.log
tail -n 2 gpurun_out/r02r_ref.log

set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02n_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_scan_tc.py tests/test_gpu_parity.py -x -q > gpurun_out/r02n_pytest.log 2>&1; tail -n 2 gpurun_out/r02n_pytest.log
timeout 1200 python bench.py --lat-calls 0 --no-paper-timing --no-cpu-baseline --modes greedy --and-scan 2000,50000 > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.log; tail -n 1 gpurun_out/r02n_bench.log
timeout 900 scripts/profile.sh launches r02n --no-paper-timing --steps 2 --warmup 3 --modes greedy --and-scan 2000 --widths 2
python scripts/summarize_profile.py gpurun_out/r02n_ncu.md --launches gpurun_out/r02n_launches.csv > /dev/null 2>&1; head -16 gpurun_out/r02n_ncu.md

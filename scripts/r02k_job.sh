set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02k_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_scan_tc.py tests/test_gpu_parity.py -x -q > gpurun_out/r02k_pytest.log 2>&1; tail -n 2 gpurun_out/r02k_pytest.log
timeout 1200 python bench.py --lat-calls 0 --no-paper-timing --no-cpu-baseline --modes greedy --and-scan 2000,50000 > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.log
timeout 1200 python bench.py --config sift --lat-calls 0 --no-cpu-baseline > gpurun_out/r02k_bench_sift.json 2> gpurun_out/r02k_bench_sift.log
timeout 900 scripts/profile.sh launches r02k --no-paper-timing --steps 2 --warmup 3 --modes greedy --and-scan 2000 --widths 2
NCU_COUNT=4 timeout 1500 scripts/profile.sh full r02k "k_scan_tc|k_and_filter|k_pack" --no-paper-timing --steps 1 --warmup 3 --modes greedy --and-scan 2000 --widths 2
python scripts/summarize_profile.py gpurun_out/r02k_ncu.md --launches gpurun_out/r02k_launches.csv --full gpurun_out/r02k_full.ncu-rep > /dev/null 2>&1

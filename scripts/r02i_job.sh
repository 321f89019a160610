set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02i_build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_graph_build.py -x -q > gpurun_out/r02i_pytest_gb.log 2>&1; tail -n 3 gpurun_out/r02i_pytest_gb.log
timeout 300 python scripts/prof_builder.py --points 2000000 > gpurun_out/r02i_builder.log 2>&1; tail -n 2 gpurun_out/r02i_builder.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scan_tc.py tests/test_gpu_small.py -x -q > gpurun_out/r02i_pytest.log 2>&1; tail -n 3 gpurun_out/r02i_pytest.log
timeout 1200 python bench.py --lat-calls 100 --no-paper-timing > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.log; grep -v "greedy\|parallel" gpurun_out/r02i_bench.log | tail -n 4 | cut -c1-300

set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02j_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_scan_tc.py tests/test_gpu_graph_build.py tests/test_gpu_parity.py tests/test_gpu_small.py -x -q > gpurun_out/r02j_pytest.log 2>&1; tail -n 3 gpurun_out/r02j_pytest.log
timeout 1200 python bench.py --lat-calls 100 --no-paper-timing > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.log; grep -v "greedy\|parallel" gpurun_out/r02j_bench.log | tail -n 3 | cut -c1-300
VF_PACK=0 timeout 1200 python bench.py --lat-calls 0 --no-paper-timing --no-cpu-baseline --modes greedy --and-scan 2000 --widths 2 > gpurun_out/r02j_bench_nopack.json 2> gpurun_out/r02j_bench_nopack.log
timeout 1200 python bench.py --config sift --lat-calls 0 --no-cpu-baseline > gpurun_out/r02j_bench_sift.json 2> gpurun_out/r02j_bench_sift.log

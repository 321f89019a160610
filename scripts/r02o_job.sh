set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02o_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_scan_tc.py tests/test_gpu_parity.py tests/test_gpu_small.py -x -q > gpurun_out/r02o_pytest.log 2>&1; tail -n 2 gpurun_out/r02o_pytest.log
timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 2000 VF_GRAPH_FIRST=0 VF_GRAPH_FIRST=1 VF_GRAPH_FIRST=1,VF_GRAPH_PER_SM=2 VF_GRAPH_FIRST=1,VF_GRAPH_PER_SM=4 VF_OVERLAP=0 > gpurun_out/r02o_ab.log 2>&1; cat gpurun_out/r02o_ab.log | grep step
timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 VF_GRAPH_FIRST=0 VF_GRAPH_FIRST=1 > gpurun_out/r02o_ab99.log 2>&1; grep step gpurun_out/r02o_ab99.log
NCU_COUNT=2 timeout 1500 scripts/profile.sh full r02o "k_and_filter|k_graph" --no-paper-timing --steps 1 --warmup 3 --modes greedy --and-scan 50000 --widths 2 --targets 0.99
python scripts/summarize_profile.py gpurun_out/r02o_ncu.md --full gpurun_out/r02o_full.ncu-rep > /dev/null 2>&1

set -u
mkdir -p gpurun_out
export VF_GRAPH_CACHE=/tmp/vf_graph_cache
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02q_build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "search_width or single_label or multilabel or overflow" > gpurun_out/r02q_pytest.log 2>&1; tail -n 2 gpurun_out/r02q_pytest.log
timeout 900 python scripts/ab_env.py --config yfcc --itopk 192 --w 2 --and-scan 50000 VF_GRAPH_WARP_KB=7 VF_GRAPH_WARP_KB=10 VF_GRAPH_WARP_KB=14 VF_GRAPH_WARP_KB=20 VF_GRAPH_WARP_KB=28 > gpurun_out/r02q_ab192.log 2>&1; grep step gpurun_out/r02q_ab192.log
timeout 900 python scripts/ab_env.py --config yfcc --itopk 32 --w 2 --and-scan 2000 VF_GRAPH_WARP_KB=7 VF_GRAPH_WARP_KB=10 VF_GRAPH_WARP_KB=14 > gpurun_out/r02q_ab32.log 2>&1; grep step gpurun_out/r02q_ab32.log
timeout 900 python scripts/ab_env.py --config sift --itopk 48 --w 2 VF_GRAPH_WARP_KB=7 VF_GRAPH_WARP_KB=10 VF_GRAPH_WARP_KB=14 > gpurun_out/r02q_absift.log 2>&1; grep step gpurun_out/r02q_absift.log
VF_NVCC_EXTRA=-DVF_TC_PROF timeout 900 python scripts/tc_prof.py --config yfcc --itopk 32 --and-scan 2000 --reps 1 > gpurun_out/r02q_tcprof.log 2>&1
python -c "from paper_2506_00812_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
grep "TCPROF blk 0" gpurun_out/r02q_tcprof.log | tail -n 6

set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python scripts/prof_builder.py --points 300000 > gpurun_out/r02h_builder.log 2>&1
timeout 900 ncu --set full --import-source on -k regex:k_join -c 1 -o gpurun_out/r02h_join python scripts/prof_builder.py --points 300000 > gpurun_out/r02h_join.log 2>&1
tail -3 gpurun_out/r02h_builder.log gpurun_out/r02h_join.log
timeout 600 python -m pytest tests/test_gpu_scan_tc.py tests/test_gpu_parity.py -x -q > gpurun_out/r02h_pytest.log 2>&1; tail -3 gpurun_out/r02h_pytest.log
VF_NVCC_EXTRA=-DVF_TC_PROF timeout 900 python scripts/tc_prof.py --config yfcc --itopk 32 --and-scan 2000 --reps 2 > gpurun_out/r02h_tcprof.log 2>&1
grep TCPROF gpurun_out/r02h_tcprof.log | tail -8

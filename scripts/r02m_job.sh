set -u
mkdir -p gpurun_out
VF_NVCC_EXTRA=-DVF_TC_PROF timeout 900 python scripts/tc_prof.py --config yfcc --itopk 32 --and-scan 2000 --reps 1 > gpurun_out/r02m_tcprof.log 2>&1
python -c "from paper_2506_00812_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
grep -c TCBIG gpurun_out/r02m_tcprof.log; grep TCBIG gpurun_out/r02m_tcprof.log | sort -t' ' -k6 -n -r | head -n 20
timeout 900 python -m pytest tests/test_gpu_scan_tc.py tests/test_gpu_parity.py -x -q > gpurun_out/r02m_pytest.log 2>&1; tail -n 2 gpurun_out/r02m_pytest.log
timeout 1200 python bench.py --lat-calls 0 --no-paper-timing --no-cpu-baseline --modes greedy --and-scan 2000,50000 > gpurun_out/r02m_bench.json 2> gpurun_out/r02m_bench.log; tail -n 1 gpurun_out/r02m_bench.log

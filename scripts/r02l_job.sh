set -u
mkdir -p gpurun_out
VF_NVCC_EXTRA=-DVF_TC_PROF timeout 900 python scripts/tc_prof.py --config yfcc --itopk 32 --and-scan 2000 --reps 2 > gpurun_out/r02l_tcprof.log 2>&1
python -c "from paper_2506_00812_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
grep TCPROF gpurun_out/r02l_tcprof.log | tail -n 6

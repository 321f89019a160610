set -u
mkdir -p gpurun_out
VF_NVCC_EXTRA=-DVF_TC_PROF timeout 900 python scripts/tc_prof.py --config yfcc --itopk 32 --and-scan 2000 --reps 2 > gpurun_out/r02g_tcprof.log 2>&1
python -c "from paper_2506_00812_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
timeout 600 python scripts/prof_builder.py --points 2000000 > gpurun_out/r02g_builder.log 2>&1
timeout 900 ncu --set full --import-source on -k regex:k_join -c 2 -o gpurun_out/r02g_join python scripts/prof_builder.py --points 2000000 > gpurun_out/r02g_join.log 2>&1
tail -3 gpurun_out/r02g_builder.log; grep -c TCPROF gpurun_out/r02g_tcprof.log

set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
bash scripts/r02_sanitize.sh r02p
timeout 2400 python scripts/f2_sweep.py > gpurun_out/r02p_f2.json 2> gpurun_out/r02p_f2.log; echo "f2 rc=$?"; tail -n 12 gpurun_out/r02p_f2.log

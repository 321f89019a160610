#!/bin/bash
# compute-sanitizer on tiny inputs (scripts/sanitize.py): memcheck, racecheck, synccheck, initcheck.
# Logs -> gpurun_out/<tag>_san_<tool>.log
set -u
tag=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize.py > gpurun_out/${tag}_san_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/${tag}_san_${tool}.log
  tail -n 4 gpurun_out/${tag}_san_${tool}.log
done

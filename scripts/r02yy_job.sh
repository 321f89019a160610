#!/bin/bash
# full-size parity incl. the 10M YFCC-shaped test at the final operating points
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02yy_build.log 2>&1 || exit 1
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -m gpu -v > gpurun_out/r02yy_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02yy_pytest.log; grep -E "PASS|FAIL|rc=" gpurun_out/r02yy_pytest.log | tail -n 14

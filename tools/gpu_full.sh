#!/bin/bash
# full GPU test suite + smoke + one ncu capture of the row-split kernel (config 2, 2 ranks in one grid)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_rs -s 1 -c 1 -o gpurun_out/k_pcg_rs_full python tools/rowsplit_rate.py 2 > gpurun_out/ncu_rs.log 2>&1; echo "ncu rc $?"; tail -2 gpurun_out/ncu_rs.log

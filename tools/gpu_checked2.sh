# the bounds-checked build on the grouped layout (and with replicas on): GPU suite + small-size driver
bash tools/gpu_checked.sh
export PCGS_LIBRARY=$PWD/paper_1810_12437_b200/libpcgs_checked.so
PCGS_REPLICAS=1 timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_cg.py tests/test_gpu_rowsplit.py tests/test_gpu_gibbs.py -q -k "not config2 and not parity" > gpurun_out/pytest_checked_rep.log 2>&1; echo "checked+replicas pytest rc $?"
tail -2 gpurun_out/pytest_checked_rep.log
grep -c "pcgs check failed" gpurun_out/pytest_checked_rep.log

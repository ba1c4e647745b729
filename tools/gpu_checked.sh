# GPU suite against the bounds-checked library (PCGS_CHECKED=1): the substitute
# for compute-sanitizer, which is closed on this pool
mkdir -p gpurun_out
export PCGS_LIBRARY=$PWD/paper_1810_12437_b200/libpcgs_checked.so
timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_cg.py tests/test_gpu_sampler.py tests/test_gpu_rowsplit.py tests/test_gpu_batched.py tests/test_gpu_batched_gibbs.py tests/test_gpu_affine.py tests/test_gpu_gibbs.py tests/test_gpu_diagnostics.py -q -rf -k "not config2 and not parity" > gpurun_out/pytest_checked.log 2>&1; echo "checked pytest rc $?"
tail -5 gpurun_out/pytest_checked.log
grep -c "pcgs check failed" gpurun_out/pytest_checked.log
timeout 300 python tools/sanitize_small.py > gpurun_out/sanitize_small_checked.log 2>&1; echo "sanitize_small (checked) rc $?"; tail -2 gpurun_out/sanitize_small_checked.log

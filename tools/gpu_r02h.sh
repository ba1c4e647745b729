mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_affine.py tests/test_gpu_dropin.py tests/test_gpu_sparse.py tests/test_gpu_cg.py tests/test_gpu_sampler.py tests/test_gpu_gibbs.py -q -rf -s > gpurun_out/pytest_h.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|FAILED|Error|z-scores" gpurun_out/pytest_h.log | tail -30
timeout 600 python tools/batched_rate.py --iters 100 --R 1 > gpurun_out/r1.jsonl 2>&1; cut -c1-120 gpurun_out/r1.jsonl

mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_rowsplit.py tests/test_gpu_rowsplit_gibbs.py tests/test_gpu_sampler.py tests/test_gpu_gibbs.py -q -rf -s > gpurun_out/pytest_b.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|z-scores|rel L2|Error" gpurun_out/pytest_b.log | tail -30
timeout 900 python bench.py --steps 20 --warmup 5 --record > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err; echo "bench rc $?"
cat gpurun_out/bench_b.json; tail -5 gpurun_out/bench_b.err

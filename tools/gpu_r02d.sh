mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batched.py -q -rf -x -s > gpurun_out/pytest_batched.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|chain [0-9]|Error|error" gpurun_out/pytest_batched.log | tail -30
timeout 600 python tools/batched_rate.py --iters 100 > gpurun_out/batched_rate.jsonl 2> gpurun_out/batched_rate.err; echo "rate rc $?"
cat gpurun_out/batched_rate.jsonl | cut -c1-200; tail -3 gpurun_out/batched_rate.err

mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -q -rf --durations=8 > gpurun_out/pytest_gpu_head.log 2>&1 ) 2>&1 | grep real; echo "pytest rc $?"
grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu_head.log | tail -8

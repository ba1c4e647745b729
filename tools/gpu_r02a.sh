mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python tools/parity_config2.py > gpurun_out/parity.jsonl 2> gpurun_out/parity.err; echo "parity rc $?"
cat gpurun_out/parity.jsonl

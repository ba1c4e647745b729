mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_batched_gibbs.py -q -rf -s > gpurun_out/pytest_k.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|FAILED|Error|z-scores" gpurun_out/pytest_k.log | tail -12
for K in 20 60; do timeout 900 python tools/fused_rate.py $K > gpurun_out/fused_rate_$K.json 2>&1; cut -c1-260 gpurun_out/fused_rate_$K.json; done

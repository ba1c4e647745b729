mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_batched_gibbs.py tests/test_gpu_gibbs.py -q -rf -x -s -k "batched or fused or run_chains" > gpurun_out/pytest_j.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|FAILED|Error|error|z-scores|Mismatch|max" gpurun_out/pytest_j.log | tail -25
timeout 900 python bench.py --workload config4 --steps 10 --warmup 3 > gpurun_out/c4_fused.json 2> gpurun_out/c4_fused.err; echo "c4 fused rc $?"
python -c "import json; d=json.load(open('gpurun_out/c4_fused.json')); print(d['value'], d['ms_per_step'], d['extra'])"; tail -3 gpurun_out/c4_fused.err

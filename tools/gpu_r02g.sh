mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_batched_gibbs.py tests/test_gpu_gibbs.py -q -rf -x -s -k "batched or run_chains or concurrent" > gpurun_out/pytest_g.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|Error|error|z-scores" gpurun_out/pytest_g.log | tail -20
timeout 900 python bench.py --workload config4 --steps 6 --warmup 3 > gpurun_out/c4_batched.json 2> gpurun_out/c4_batched.err; echo "c4 batched rc $?"
python -c "import json; d=json.load(open('gpurun_out/c4_batched.json')); print(d['value'], d['ms_per_step'], d['extra'])"; tail -3 gpurun_out/c4_batched.err
timeout 900 python bench.py --workload config4 --steps 6 --warmup 3 --concurrent 4 > gpurun_out/c4_slots.json 2> gpurun_out/c4_slots.err; echo "c4 slots rc $?"
python -c "import json; d=json.load(open('gpurun_out/c4_slots.json')); print(d['value'], d['ms_per_step'], d['extra'])"; tail -3 gpurun_out/c4_slots.err

# validation of the current build: GPU suite, smoke, bench (both arms)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
( time timeout 2400 python -m pytest tests -m gpu -x -q -rf --durations=15 > gpurun_out/pytest_gpu_head.log 2>&1 ) 2>&1 | grep real; echo "pytest rc $?"
grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu_head.log | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
( time timeout 900 python bench.py > gpurun_out/bench_head.json 2> gpurun_out/bench_head.err ) 2>&1 | grep real; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/bench_head.json')); print(d['value'], d['e2e']['value'], d['roofline']['us_per_apply'], d['roofline']['frac'], d['extra']['full_run']['iter_per_s'], d['clocks'])"

mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -rf --durations=12 -s > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu_full.log | tail -8
grep -E "^seed [0-9]|chain [0-9] \(fixture|race:" gpurun_out/pytest_gpu_full.log | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/bench_r02.json')); print(d['value'], d['e2e']['value'], d['roofline']['us_per_apply'], d['roofline']['frac'], d['extra']['full_run']['iter_per_s'], d['clocks'])"
timeout 900 python bench.py --workload config4 --steps 10 --warmup 3 > gpurun_out/bench_c4_r02.json 2> gpurun_out/bench_c4_r02.err; echo "c4 rc $?"
python -c "import json; d=json.load(open('gpurun_out/bench_c4_r02.json')); print(d['value'], d['ms_per_step'], d['extra'])"
bash tools/gpu_c4modes.sh 20 > gpurun_out/c4modes.txt 2>&1; cat gpurun_out/c4modes.txt
timeout 1200 python bench.py --workload config5 --steps 3 --warmup 1 > gpurun_out/bench_c5_r02.json 2> gpurun_out/bench_c5_r02.err; echo "c5 rc $?"
python -c "import json; d=json.load(open('gpurun_out/bench_c5_r02.json')); print(d['value'], d['ms_per_step'], d.get('roofline'))" 2>&1 | cut -c1-300
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02.json 2> gpurun_out/bench_ref_r02.err; echo "ref rc $?"; cut -c1-400 gpurun_out/bench_ref_r02.json

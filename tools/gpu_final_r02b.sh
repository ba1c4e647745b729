# round-2 evidence after the grouped pass layout: GPU suite, smoke, bench (all workloads), launch list, ncu capture of k_pcg
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
( time timeout 2400 python -m pytest tests -m gpu -x -q -rf --durations=8 > gpurun_out/pytest_gpu_r02b.log 2>&1 ) 2>&1 | grep real; echo "pytest rc $?"
grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu_r02b.log | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 --record > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/bench_r02b.json')); print(d['value'], d['e2e']['value'], d['roofline']['us_per_apply'], d['roofline']['frac'], d['extra']['full_run']['iter_per_s'], d['clocks'])"
timeout 900 python bench.py > gpurun_out/bench_default_r02b.json 2> gpurun_out/bench_default_r02b.err; echo "bench default rc $?"
timeout 900 python bench.py --workload config1 > gpurun_out/bench_config1_r02b.json 2>/dev/null; echo "c1 rc $?"
timeout 900 python bench.py --prior bridge > gpurun_out/bench_bridge_r02b.json 2>/dev/null; echo "bridge rc $?"
bash tools/gpu_c4modes.sh 20 > gpurun_out/c4modes_r02b.txt 2>&1; cat gpurun_out/c4modes_r02b.txt
timeout 1500 python bench.py --workload config5 --steps 3 --warmup 1 > gpurun_out/bench_c5_r02b.json 2> gpurun_out/bench_c5_r02b.err; echo "c5 rc $?"
python -c "import json; d=json.load(open('gpurun_out/bench_c5_r02b.json')); print(d['value'], d['ms_per_step'], d.get('roofline'))" 2>&1 | cut -c1-300
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r02b.json 2> gpurun_out/bench_ref_r02b.err; echo "ref rc $?"; cut -c1-300 gpurun_out/bench_ref_r02b.json
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-full-run"
$B > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r02b.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc $?"
C="python tools/batched_rate.py --R 1 --iters 30 --reps 1"
$C > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pcg -c 1 -o gpurun_out/k_pcg_r02b $C > gpurun_out/ncu_kpcg.log 2>&1
echo "k_pcg capture rc $?"
python tools/pass_phases.py 2>&1 | tail -2
python tools/sync_times_pcg.py 2>&1 | tail -5
python tools/rowsplit_rate.py 2>&1 | tail -8

# final round-2 evidence: GPU suite, smoke, bench, config 4, launch list, ncu captures of k_pcg and k_spcg<8>
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -rf -s > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu_final.log | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/bench_final.json')); print(d['value'], d['e2e']['value'], d['roofline']['us_per_apply'], d['roofline']['frac'], d['extra']['full_run']['iter_per_s'], d['clocks'])"
bash tools/gpu_c4modes.sh 20 > gpurun_out/c4modes_final.txt 2>&1; cat gpurun_out/c4modes_final.txt
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-full-run"
$B > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_final.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc $?"
C="python tools/batched_rate.py --R 1 --iters 30 --reps 1"
$C > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pcg -c 1 -o gpurun_out/k_pcg_final $C > gpurun_out/ncu_kpcg.log 2>&1
echo "k_pcg capture rc $?"
C2="python tools/batched_rate.py --R 8 --iters 20 --reps 1"
$C2 > gpurun_out/ncu_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spcg -c 1 -o gpurun_out/k_spcg8_final $C2 > gpurun_out/ncu_kspcg.log 2>&1
echo "k_spcg capture rc $?"

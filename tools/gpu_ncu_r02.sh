mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-full-run"
$B > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r02.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc $?"
C="python tools/batched_rate.py --R 1 --iters 30 --reps 1"
$C > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pcg -c 1 -o gpurun_out/k_pcg_r02 $C > gpurun_out/ncu_kpcg.log 2>&1
echo "k_pcg capture rc $?"; tail -2 gpurun_out/ncu_kpcg.log

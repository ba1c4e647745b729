mkdir -p gpurun_out
C="python tools/batched_rate.py --R 1 --iters 30 --reps 1"
$C > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pcg -c 1 -o gpurun_out/k_pcg_group $C > gpurun_out/ncu_kpcg.log 2>&1
echo "k_pcg capture rc $?"; tail -2 gpurun_out/ncu_kpcg.log; cat gpurun_out/ncu_plain2.log | tail -2

mkdir -p gpurun_out
CMD="python tools/batched_rate.py --R 8 --iters 20 --reps 1"
$CMD > gpurun_out/ncu_b_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spcg -c 1 -o gpurun_out/k_spcg8 $CMD > gpurun_out/ncu_b.log 2>&1
echo "ncu rc $?"; tail -3 gpurun_out/ncu_b.log

# config 4 modes at the same scans (K), the same chains: sequential, slots, batched scan-by-scan, fused
mkdir -p gpurun_out
K=${1:-20}
for m in "--config4-sequential" "--concurrent 4" "" "--config4-fused"; do
  timeout 1500 python bench.py --workload config4 --steps $K --warmup 3 $m > gpurun_out/c4mode.json 2> gpurun_out/c4mode.err
  python -c "import json; d=json.load(open('gpurun_out/c4mode.json')); print('$m', round(d['value'],1), d['config']['mode'], round(d['ms_per_step'],2), round(d['extra']['cg_iters_mean'],1))"
done

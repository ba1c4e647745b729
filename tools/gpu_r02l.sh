mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_batched_gibbs.py -q -rf -x -k "not fused_posterior" > gpurun_out/pytest_l.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_l.log
for lib in libpcgs.so libpcgs_single.so; do
  PCGS_LIBRARY=$PWD/paper_1810_12437_b200/$lib timeout 300 python tools/batched_rate.py --iters 100 --R 8,4,2 --profile > gpurun_out/rate_$lib.jsonl 2>&1
  python -c "
import json
for l in open('gpurun_out/rate_$lib.jsonl'):
    if l.startswith('{'): d=json.loads(l); print('$lib', d['R'], round(d['us_per_chain_iteration'],2), {k: round(v,1) for k,v in d['store'].get('phases_us',{}).items()})
"
done

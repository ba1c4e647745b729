mkdir -p gpurun_out
for lib in libpcgs.so libpcgs_pipe4.so libpcgs_u2.so libpcgs_u6.so; do
  PCGS_LIBRARY=$PWD/paper_1810_12437_b200/$lib timeout 300 python tools/batched_rate.py --iters 100 --R 8 --profile > gpurun_out/rate_$lib.jsonl 2>&1; echo "$lib rc $?"
  python -c "
import json,sys
for l in open('gpurun_out/rate_$lib.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['R'], round(d['us_per_chain_iteration'],2), d['store'].get('phases_us'))
"
done

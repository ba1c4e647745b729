mkdir -p gpurun_out
for lib in libpcgs.so libpcgs_l1next.so libpcgs_l1next_dist8.so libpcgs_ring4.so libpcgs.so; do
  PCGS_LIBRARY=$PWD/paper_1810_12437_b200/$lib timeout 300 python tools/batched_rate.py --iters 150 --R 1 --reps 5 > gpurun_out/ab_$lib.jsonl 2>&1
  python -c "
import json
for l in open('gpurun_out/ab_$lib.jsonl'):
    if l.startswith('{'): d=json.loads(l); print('$lib', round(d['us_per_apply'],2))
"
done

# A/B of library variants given as tags (libpcgs_TAG.so): k_pcg us per apply at config 2
mkdir -p gpurun_out
for tag in "$@"; do
  PCGS_LIBRARY=$PWD/paper_1810_12437_b200/libpcgs_$tag.so timeout 300 python tools/batched_rate.py --iters 150 --R 1 --reps 5 > gpurun_out/sw_$tag.jsonl 2>&1
  python -c "
import json
for l in open('gpurun_out/sw_$tag.jsonl'):
    if l.startswith('{'): d=json.loads(l); print('$tag', round(d['us_per_apply'],2))
"
done

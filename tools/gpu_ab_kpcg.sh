# A/B of single-chain k_pcg builds (tools/build_variant.py): us per Phi-apply at config 2
mkdir -p gpurun_out
for lib in "$@"; do
  PCGS_LIBRARY=$PWD/paper_1810_12437_b200/$lib timeout 300 python tools/batched_rate.py --iters 150 --R 1 --reps 5 > gpurun_out/abk_$lib.jsonl 2>&1
  python -c "
import json
for l in open('gpurun_out/abk_$lib.jsonl'):
    if l.startswith('{'): d=json.loads(l); print('$lib', round(d['us_per_apply'],2))
"
done

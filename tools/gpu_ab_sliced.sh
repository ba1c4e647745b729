# A/B of sliced-store lane mappings (tools/build_variant.py): per chain-iteration of the batched PCG
mkdir -p gpurun_out
for lib in "$@"; do
  PCGS_LIBRARY=$PWD/paper_1810_12437_b200/$lib timeout 300 python tools/batched_rate.py --iters 100 --R 8,4 --profile > gpurun_out/ab_$lib.jsonl 2>&1
  python -c "
import json
for l in open('gpurun_out/ab_$lib.jsonl'):
    if l.startswith('{'): d=json.loads(l); ph=d['store'].get('phases_us',{}); print('$lib', d['R'], round(d['us_per_chain_iteration'],2), round(ph.get('iteration',0)/d['R'],2), {k: round(v,1) for k,v in ph.items()})
"
done

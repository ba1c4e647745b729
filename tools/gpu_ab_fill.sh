mkdir -p gpurun_out
run() {  # tag lib env...
  tag=$1; lib=$2; shift 2
  env "$@" PCGS_LIBRARY=$PWD/paper_1810_12437_b200/$lib timeout 300 python tools/batched_rate.py --iters 150 --R 1 --reps 5 > gpurun_out/sw_$tag.jsonl 2>&1
  python -c "
import json
for l in open('gpurun_out/sw_$tag.jsonl'):
    if l.startswith('{'): d=json.loads(l); print('$tag', round(d['us_per_apply'],2))
"
}
for t in t8 t6 t4 t2 t0 t8c8; do run $t libpcgs_$t.so A=1; done

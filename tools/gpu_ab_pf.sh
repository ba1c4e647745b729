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
run dflt libpcgs.so A=1
for t in pf4 pf6 pf12 pf16; do run $t libpcgs_$t.so A=1; done
run dflt libpcgs.so A=1
timeout 300 python tools/sync_times_pcg.py > gpurun_out/sync_times_new.txt 2>&1; tail -5 gpurun_out/sync_times_new.txt
python tools/pass_phases.py 2>&1 | tail -2

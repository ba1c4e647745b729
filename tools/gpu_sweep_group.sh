# grouped layout tuning: library variants and builder thresholds, us per Phi-apply of k_pcg at config 2
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
run g2 libpcgs_g2.so A=1
run g3 libpcgs_g3.so A=1
run g4 libpcgs_g4.so A=1
run g2p8 libpcgs_g2p8.so A=1
run w48 libpcgs_g2.so PCGS_GW8=48 PCGS_GW4=20 PCGS_GW2=8
run w32p64 libpcgs_g2.so PCGS_GW8=32 PCGS_GW4=12 PCGS_GW2=4 PCGS_PIECE_MAX=64
run w128 libpcgs_g2.so PCGS_GW8=128 PCGS_GW4=64 PCGS_GW2=16
run p256 libpcgs_g2.so PCGS_PIECE_MAX=256
run p64 libpcgs_g2.so PCGS_PIECE_MAX=64
run close0 libpcgs_g2.so PCGS_G_CLOSE16=0 PCGS_G_SLICE_COST=0
run close2 libpcgs_g2.so PCGS_G_CLOSE16=32 PCGS_G_SLICE_COST=2
PCGS_LIBRARY=$PWD/paper_1810_12437_b200/libpcgs_g2.so timeout 300 python tools/sync_times_pcg.py > gpurun_out/sync_times_g2.txt 2>&1; tail -12 gpurun_out/sync_times_g2.txt

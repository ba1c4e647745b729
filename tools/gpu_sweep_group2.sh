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
run w128p256 libpcgs_g2.so PCGS_GW8=128 PCGS_GW4=64 PCGS_GW2=16 PCGS_PIECE_MAX=256
run w256 libpcgs_g2.so PCGS_GW8=256 PCGS_GW4=128 PCGS_GW2=32
run w256p256 libpcgs_g2.so PCGS_GW8=256 PCGS_GW4=128 PCGS_GW2=32 PCGS_PIECE_MAX=256
run no8 libpcgs_g2.so PCGS_GW8=100000 PCGS_GW4=64 PCGS_GW2=16
run no8p256 libpcgs_g2.so PCGS_GW8=100000 PCGS_GW4=64 PCGS_GW2=16 PCGS_PIECE_MAX=256
run max2 libpcgs_g2.so PCGS_GW8=100000 PCGS_GW4=100000 PCGS_GW2=32
run max2p256 libpcgs_g2.so PCGS_GW8=100000 PCGS_GW4=100000 PCGS_GW2=32 PCGS_PIECE_MAX=256
run w128g4 libpcgs_g4.so PCGS_GW8=128 PCGS_GW4=64 PCGS_GW2=16
run w128p8 libpcgs_g2p8.so PCGS_GW8=128 PCGS_GW4=64 PCGS_GW2=16

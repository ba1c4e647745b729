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
run np2 libpcgs_np2.so A=1
run p2 libpcgs_p2.so A=1
run p2_norep libpcgs_p2.so PCGS_REPLICAS=0
run p1 libpcgs_p1.so A=1
run p3 libpcgs_p3.so A=1
run p2f16 libpcgs_p2f16.so A=1
PCGS_LIBRARY=$PWD/paper_1810_12437_b200/libpcgs_p2.so timeout 600 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_cg.py -m gpu -x -q 2>&1 | tail -2

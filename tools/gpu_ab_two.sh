# A/B of two library builds (libpcgs.so vs libpcgs_prev.so): k_pcg us per apply at config 2, parity subset
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
run new libpcgs.so A=1
run prev libpcgs_prev.so A=1
run new libpcgs.so A=1
run prev libpcgs_prev.so A=1
timeout 300 python tools/sync_times_pcg.py > gpurun_out/sync_times_new.txt 2>&1; tail -5 gpurun_out/sync_times_new.txt
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_cg.py tests/test_gpu_rowsplit.py tests/test_gpu_gibbs.py -m gpu -x -q 2>&1 | tail -2

# A/B of two library builds (libpcgs.so vs libpcgs_prev.so): k_pcg us per apply at config 2, phases, parity subset
mkdir -p gpurun_out
run() {  # tag lib
  tag=$1; lib=$2
  PCGS_LIBRARY=$PWD/paper_1810_12437_b200/$lib timeout 300 python tools/batched_rate.py --iters 150 --R 1 --reps 5 > gpurun_out/sw_$tag.jsonl 2>&1
  python -c "
import json
for l in open('gpurun_out/sw_$tag.jsonl'):
    if l.startswith('{'): d=json.loads(l); print('$tag', round(d['us_per_apply'],2))
"
}
run new libpcgs.so
run prev libpcgs_prev.so
run new libpcgs.so
run prev libpcgs_prev.so
timeout 300 python tools/sync_times_pcg.py > gpurun_out/sync_times_new.txt 2>&1; tail -5 gpurun_out/sync_times_new.txt
timeout 1200 python -m pytest tests/test_gpu_cg.py tests/test_gpu_gibbs.py tests/test_gpu_parity_config2.py tests/test_gpu_affine.py tests/test_gpu_sampler.py -m gpu -x -q 2>&1 | tail -2

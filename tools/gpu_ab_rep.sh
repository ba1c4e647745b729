mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_cg.py tests/test_gpu_sampler.py tests/test_gpu_rowsplit.py tests/test_gpu_affine.py -m gpu -x -q > gpurun_out/pytest_layout.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_layout.log
run() {  # tag env...
  tag=$1; shift 1
  env "$@" timeout 300 python tools/batched_rate.py --iters 150 --R 1 --reps 5 > gpurun_out/sw_$tag.jsonl 2>&1
  python -c "
import json
for l in open('gpurun_out/sw_$tag.jsonl'):
    if l.startswith('{'): d=json.loads(l); print('$tag', round(d['us_per_apply'],2))
"
}
run rep A=1
run norep PCGS_REPLICAS=0
run rep_w48 PCGS_GW8=48 PCGS_GW4=20 PCGS_GW2=8
run rep_w80p128 PCGS_GW8=80 PCGS_GW4=40 PCGS_GW2=12 PCGS_PIECE_MAX=128
run rep_w256 PCGS_GW8=256 PCGS_GW4=128 PCGS_GW2=32
timeout 300 python tools/sync_times_pcg.py > gpurun_out/sync_times_rep.txt 2>&1; tail -5 gpurun_out/sync_times_rep.txt

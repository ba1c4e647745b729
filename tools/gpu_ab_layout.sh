# grouped vs flat pass layout (PCGS_LAYOUT): parity subset, then us per Phi-apply of k_pcg at config 2
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_cg.py tests/test_gpu_sampler.py tests/test_gpu_rowsplit.py tests/test_gpu_affine.py -m gpu -x -q > gpurun_out/pytest_layout.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_layout.log
for lay in group flat group flat; do
  PCGS_LAYOUT=$lay timeout 300 python tools/batched_rate.py --iters 150 --R 1 --reps 5 > gpurun_out/ab_layout_$lay.jsonl 2>&1
  python -c "
import json
for l in open('gpurun_out/ab_layout_$lay.jsonl'):
    if l.startswith('{'): d=json.loads(l); print('$lay', round(d['us_per_apply'],2))
"
done

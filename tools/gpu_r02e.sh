mkdir -p gpurun_out
for lib in libpcgs.so libpcgs_u2.so; do
  PCGS_LIBRARY=$PWD/paper_1810_12437_b200/$lib timeout 300 python tools/batched_rate.py --iters 100 --R 8,4 > gpurun_out/rate_$lib.jsonl 2>&1; echo "$lib rc $?"
  cut -c1-140 gpurun_out/rate_$lib.jsonl
done
timeout 900 python -m pytest tests/test_gpu_batched.py tests/test_gpu_race.py -q -rf -x -s > gpurun_out/pytest_e.log 2>&1; echo "pytest rc $?"
grep -E "passed|failed|chain [0-9]|race:|Error" gpurun_out/pytest_e.log | tail -20

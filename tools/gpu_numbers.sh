#!/bin/bash
# the secondary measurements quoted in DESIGN.md (config 2 PCG variants, config 4 and 5 runs)
mkdir -p gpurun_out
timeout 600 python tools/rowsplit_rate.py 2>&1 | tail -5
timeout 600 python tools/concurrent_chains.py 2>&1 | tail -6
for R in 1 4; do timeout 600 python bench.py --workload config4 --concurrent $R --steps 6 --warmup 3 2>/dev/null | tail -1; done > gpurun_out/bench_config4.jsonl
cat gpurun_out/bench_config4.jsonl | cut -c1-100
timeout 1200 python bench.py --workload config5 --steps 6 --warmup 3 > gpurun_out/bench_config5.json 2>/dev/null; cut -c1-100 gpurun_out/bench_config5.json

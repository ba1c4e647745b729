#!/bin/bash
# bench line + ncu launch list of the bench command + one full k_pcg capture (config 2 solve)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
cat gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu1 rc $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg -s 1 -c 1 -o gpurun_out/k_pcg_full python tools/prof_pcg.py > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc $?"
tail -3 gpurun_out/ncu_full.log

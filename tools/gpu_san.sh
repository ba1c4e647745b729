# usage: bash tools/gpu_san.sh <tool>   (one compute-sanitizer tool per gpurun call)
mkdir -p gpurun_out
T=$1
timeout 600 python tools/sanitize_small.py > gpurun_out/san_plain_$T.log 2>&1; echo "plain rc $?"; tail -3 gpurun_out/san_plain_$T.log
timeout 2400 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_small.py > gpurun_out/san_$T.log 2>&1; echo "$T rc $?"
tail -25 gpurun_out/san_$T.log

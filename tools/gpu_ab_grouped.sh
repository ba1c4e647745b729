# The A/B runs behind DESIGN.md §3/§4 (grouped pass layout), in the order they were made.
# Every line is `k_pcg us per Phi-apply at config 2` from tools/batched_rate.py --iters 150 --R 1 --reps 5
# (results: profiles/layout_ab_r02b.txt).  Variants are built here first, e.g.
#   python tools/build_variant.py flat  -DPCGS_FLAT_WALK=1          (then PCGS_LAYOUT=flat|group selects the store)
#   python tools/build_variant.py pp2   -DPCGS_GPIPE=1 -DPCGS_GRING=2
#   python tools/build_variant.py np2   -DPCGS_GPIPE=0 -DPCGS_GRING=2
#   python tools/build_variant.py pf8   -DPCGS_GPREFETCH=8
# and run on the GPU box with:  gpurun -- 'bash tools/gpu_ab_grouped.sh TAG [ENV=VALUE ...] -- TAG ...'
mkdir -p gpurun_out
run() {  # tag env...
  tag=$1; shift 1
  lib=libpcgs_$tag.so; [ "$tag" = dflt ] && lib=libpcgs.so
  env "$@" PCGS_LIBRARY=$PWD/paper_1810_12437_b200/$lib timeout 300 python tools/batched_rate.py --iters 150 --R 1 --reps 5 > gpurun_out/ab_$tag.jsonl 2>&1
  python -c "
import json, sys
for l in open('gpurun_out/ab_$tag.jsonl'):
    if l.startswith('{'): d=json.loads(l); print('$tag', ' '.join(sys.argv[1:]), round(d['us_per_apply'],2))
" "$@"
}
args=()
for a in "$@"; do
  if [ "$a" = "--" ]; then run "${args[@]}"; args=(); else args+=("$a"); fi
done
[ ${#args[@]} -gt 0 ] && run "${args[@]}"
# builder knobs (environment, read when the store is built):
#   PCGS_GW8 / PCGS_GW4 / PCGS_GW2   vectors from which a segment gets an 8 / 4 / 2-lane group (128 / 64 / 16)
#   PCGS_PIECE_MAX                   vectors per CSC piece (256)
#   PCGS_G_CLOSE16, PCGS_G_SLICE_COST   cost-model charges per segment / slice (16, 1)
#   PCGS_REPLICAS=1                  replicas of hot slab entries (off)
#   PCGS_CSC_SLAB_MAX                rows per CSC slab (4 slabs at config 2; 6: 71.6 us, 8: 72.3, 12: 81.4)

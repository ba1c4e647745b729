#!/bin/bash
# PCG us/iter (config 2) for variant builds (libpcgs_v_*.so) and environment knobs
for r in 1 2; do
  echo -n "in-tree "; python tools/pcg_rate.py 0
  for f in paper_1810_12437_b200/libpcgs_v_*.so; do echo -n "$(basename $f) "; PCGS_LIBRARY=$f python tools/pcg_rate.py 0; done
  for e in ${ENVS:-}; do echo -n "$e "; env $e python tools/pcg_rate.py 0; done
done

#!/bin/bash
# A/B: PCG us/iter (config 2) of the working tree vs the HEAD build (tools/build_head_variant.py)
for r in 1 2 3; do
  echo -n "head "; PCGS_LIBRARY=paper_1810_12437_b200/libpcgs_v_head.so python tools/pcg_rate.py 0
  echo -n "new  "; python tools/pcg_rate.py 0
done

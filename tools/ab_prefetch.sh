#!/bin/bash
# A/B of prefetch-window builds (libpcgs_pf<first>_<dist>.so) vs the in-tree library
for r in 1 2; do
  for f in paper_1810_12437_b200/libpcgs_pf*.so; do echo -n "$(basename $f) "; PCGS_LIBRARY=$f python tools/pcg_rate.py 0; done
  echo -n "in-tree "; python tools/pcg_rate.py 0
done

#!/bin/bash
# A/B: PCG us/iter of the in-tree library vs an alternative build (PCGS_LIBRARY)
# usage: tools/ab_rate.sh paper_1810_12437_b200/libpcgs_base.so [rounds]
ALT=$1; N=${2:-2}
for r in $(seq 1 $N); do
  echo -n "new  "; python tools/pcg_rate.py 0
  echo -n "base "; PCGS_LIBRARY=$ALT python tools/pcg_rate.py 0
done

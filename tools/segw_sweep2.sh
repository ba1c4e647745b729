#!/bin/bash
# sweep the block / emit charges of the balancing cost model (store.cpp)
for cfg in ${CFGS:-"12 0"}; do
  set -- $cfg
  echo "== block=$1 emit=$2"
  PCGS_SEG_WEIGHT=$1 PCGS_SEG_EMIT=$2 python tools/pcg_rate.py 0
  PCGS_SEG_WEIGHT=$1 PCGS_SEG_EMIT=$2 python tools/sync_times_pcg.py 2>/dev/null | sed -n 2,4p
done

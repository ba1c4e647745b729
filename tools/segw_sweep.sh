#!/bin/bash
for w in ${WEIGHTS:-0 2 4 8 16}; do
  echo "== PCGS_SEG_WEIGHT=$w"
  PCGS_SEG_WEIGHT=$w python tools/pcg_rate.py 0
  PCGS_SEG_WEIGHT=$w python tools/sync_times_pcg.py 2>/dev/null | head -3
done

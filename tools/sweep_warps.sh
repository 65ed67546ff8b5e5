#!/bin/bash
# Block-size sweep of the fused kernel per workload (development aid).
for nw in 1 2 3 4 5 6 7 8; do
  echo "== warps/block $nw"
  UFPGD_FUSED_WARPS=$nw python tools/quick_time.py 1 2 3 2>&1 | grep cfg
done

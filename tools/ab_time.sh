#!/bin/bash
# Times the A/B library variants in tools/ablib/* on the given configs.
cfgs=${CFGS:-"1 2"}
for d in ${VARIANTS:-$(ls tools/ablib)}; do
  [ -f tools/ablib/$d/libufpgd_gpu.so ] || continue
  echo "== $d"; UFPGD_LIB=tools/ablib/$d/libufpgd_gpu.so python tools/quick_time.py $cfgs 2>&1 | grep cfg
done

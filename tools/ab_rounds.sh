#!/bin/bash
# Interleaved A/B timing of tools/ablib/* variants (development aid):
# ROUNDS x (each variant once) on CFGS, so box drift hits every variant alike.
cfgs=${CFGS:-"4 5"}
for r in $(seq ${ROUNDS:-3}); do
  for d in ${VARIANTS:-$(ls tools/ablib)}; do
    [ -f tools/ablib/$d/libufpgd_gpu.so ] || continue
    UFPGD_LIB=tools/ablib/$d/libufpgd_gpu.so QT_ROUNDS=${QT_ROUNDS:-3} python tools/quick_time.py $cfgs 2>&1 | grep cfg | sed "s/^/[$d r$r] /"
  done
done

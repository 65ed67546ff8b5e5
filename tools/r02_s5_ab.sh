#!/bin/bash
# Session-5 A/B: pair kernel at 8 CTAs/SM (p8), (16,128) at 5 CTAs/SM (m5) vs HEAD (development aid).
out=gpurun_out/s5ab; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_pair.py tests/test_gpu_parity.py -m gpu -x -q > $out/tests.log 2>&1; echo "tests rc=$?" | tee -a $out/tests.log
VARIANTS="${VARIANTS:-head p8 m5}" CFGS="${CFGS:-2 3 5}" ROUNDS=3 bash tools/ab_rounds.sh 2>&1 | tee $out/ab.log

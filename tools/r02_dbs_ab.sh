#!/bin/bash
# DBS (direct Bs build) check + A/B against the HEAD library (development aid).
out=gpurun_out/dbs; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_mma.py tests/test_gpu_pair.py tests/test_gpu_parity.py -m gpu -x -q > $out/tests.log 2>&1; echo "tests rc=$?" | tee -a $out/tests.log
tail -5 $out/tests.log
VARIANTS="${VARIANTS:-head dbs}" CFGS="2 3 5 4" ROUNDS=3 bash tools/ab_rounds.sh 2>&1 | tee $out/ab.log

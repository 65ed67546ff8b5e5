#!/bin/bash
# ncu captures of the tcgen05 kernel at HEAD + per-layer phase stamps (development aid).
out=${1:-gpurun_out/r02h}
mkdir -p $out
for c in 4 5; do
  n=$([ $c = 5 ] && echo 65536 || echo 16384)
  python tools/one_launch.py $c $n > /dev/null && \
  ncu --set full --clock-control none --import-source on -k regex:mma_kernel -s 2 -c 1 -f -o $out/ncu_mma_cfg$c python tools/one_launch.py $c $n > $out/ncu_mma_cfg$c.log 2>&1
done
if [ -f tools/ablib/timing/libufpgd_gpu.so ]; then
  UFPGD_LIB=tools/ablib/timing/libufpgd_gpu.so python tools/mma_phases.py > $out/phases.txt 2>&1
fi
echo done

#!/bin/bash
# Final round-2 ncu captures of the product kernels (development aid).
mkdir -p gpurun_out/r02f
for c in 4 5; do
  n=$([ $c = 5 ] && echo 65536 || echo 16384)
  python tools/one_launch.py $c $n > /dev/null && \
  ncu --set full --clock-control none --import-source on -k regex:mma_kernel -s 2 -c 1 -f -o gpurun_out/r02f/ncu_mma_cfg$c python tools/one_launch.py $c $n > gpurun_out/r02f/ncu_mma_cfg$c.log 2>&1
done
python tools/one_launch.py 2 > /dev/null && \
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 1 -c 1 -f -o gpurun_out/r02f/ncu_fused_cfg2 python tools/one_launch.py 2 > gpurun_out/r02f/ncu_fused_cfg2.log 2>&1
echo done

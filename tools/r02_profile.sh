#!/bin/bash
# Round-2 evidence run on the GPU box (development aid): full GPU tests, then
# ncu --set full captures of the final kernels and the bench launch list.
# Every ncu run follows a run of the same command without ncu.
set -x
mkdir -p gpurun_out/r02
python tools/one_launch.py 2 > /dev/null && \
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 1 -c 1 -f -o gpurun_out/r02/ncu_fused_cfg2 python tools/one_launch.py 2 > gpurun_out/r02/ncu_fused_cfg2.log 2>&1
python tools/one_launch.py 5 65536 > /dev/null && \
ncu --set full --clock-control none --import-source on -k regex:mma_kernel -s 2 -c 1 -f -o gpurun_out/r02/ncu_mma_cfg5 python tools/one_launch.py 5 65536 > gpurun_out/r02/ncu_mma_cfg5.log 2>&1
python tools/one_launch.py 4 > /dev/null && \
ncu --set full --clock-control none --import-source on -k regex:mma_kernel -s 2 -c 1 -f -o gpurun_out/r02/ncu_mma_cfg4 python tools/one_launch.py 4 > gpurun_out/r02/ncu_mma_cfg4.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r02/bench_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02/launches_bench_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r02/ncu_launches.log 2>&1
echo profile_done

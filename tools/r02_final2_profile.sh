#!/bin/bash
# Round-2 (session 3) evidence: smoke, ncu --set full of the three tcgen05
# product launches (config 2 pairs, configs 4 and 5) and of the FFMA2 team PGD
# kernel (config 3 shape), and the bench launch list (development aid).
out=${1:-gpurun_out/r02g}
mkdir -p $out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1
for c in 2 4 5; do
  n=$([ $c = 5 ] && echo 65536 || ([ $c = 4 ] && echo 16384 || echo 65536))
  python tools/one_launch.py $c $n > /dev/null && \
  ncu --set full --clock-control none --import-source on -k regex:mma_kernel -s 2 -c 1 -f -o $out/ncu_mma_cfg$c \
      python tools/one_launch.py $c $n > $out/ncu_mma_cfg$c.log 2>&1
done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > $out/bench_small.json 2>/dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > $out/ncu_launch.log 2>&1
echo done

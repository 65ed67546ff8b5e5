#!/bin/bash
# Session-5 final evidence: GPU tests, both bench arms, the strong-scaling mode, bench launch list.
out=${1:-gpurun_out/r02s5f}
mkdir -p $out
python -m pytest tests -m gpu -x -q > $out/gputests.log 2>&1; echo "rc=$?" >> $out/gputests.log
python bench.py --impl reference --steps 5 --warmup 1 > $out/bench_reference.json 2> $out/bench_reference.err
python bench.py > $out/bench_cfg2.json 2> $out/bench_cfg2.err
python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs > $out/bench_cfg5_strong.json 2> $out/bench_cfg5_strong.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > $out/bench_small.json 2>/dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-other-configs > $out/ncu_launch.log 2>&1
echo all-done

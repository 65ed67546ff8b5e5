#!/bin/bash
# Round-2 session-5 HEAD evidence: GPU tests, bench (both arms), smoke, ncu
# --set full of the three tcgen05 product launches, bench launch list.
out=${1:-gpurun_out/r02s5}
mkdir -p $out
python -m pytest tests -m gpu -x -q > $out/gputests.log 2>&1; echo "rc=$?" >> $out/gputests.log
python bench.py > $out/bench_cfg2.json 2> $out/bench_cfg2.err
python bench.py --impl reference --steps 5 --warmup 1 > $out/bench_reference.json 2> $out/bench_reference.err
python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs > $out/bench_cfg5_strong.json 2> $out/bench_cfg5_strong.err
bash tools/r02_final2_profile.sh $out
echo all-done

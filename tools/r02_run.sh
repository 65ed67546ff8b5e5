bash tools/r02_profile.sh > gpurun_out/r02_profile.log 2>&1
python bench.py --steps 30 --warmup 5 --cpu-seconds 10 > gpurun_out/r02/bench_full.json 2> gpurun_out/r02/bench_full.err
python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/r02/bench_cfg5.json 2> gpurun_out/r02/bench_cfg5.err
cuobjdump -sass build/obj/team.o > gpurun_out/r02/team.sass 2>/dev/null; echo all_done

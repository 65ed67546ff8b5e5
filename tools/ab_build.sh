#!/bin/bash
# Builds A/B variants of the product library into tools/ablib/<name>/ with
# extra nvcc defines (development aid): tools/ab_build.sh name -DFOO=1 ...
set -e
name=$1; shift
cd "$(dirname "$0")/.."
rm -rf build/obj/ab/$name; mkdir -p tools/ablib/$name build/obj/ab/$name
objs=""
# SRC_<name>=path overrides one source (e.g. SRC_mma=/tmp/old/mma.cu)
for f in team team64 tile mma general metrics grad datagen probe; do
  var=SRC_$f; src=${!var:-paper_2304_12745_b200/csrc/$f.cu}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC -Iinclude \
    -Ipaper_2304_12745_b200/csrc "$@" -Xptxas -v -c $src \
    -o build/obj/ab/$name/$f.o 2> build/obj/ab/$name/$f.log &
  objs="$objs build/obj/ab/$name/$f.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/ablib/$name/libufpgd_gpu.so \
  $objs build/obj/capi.o build/obj/host_gen.o build/obj/api.o build/obj/dataset_io.o build/obj/host_util.o -ldl -lpthread
grep -A2 "${AB_GREP:-fused_kernelINS0_4TeamILi8ELi64}" build/obj/ab/$name/${AB_LOG:-team}.log | grep -oE "Used [0-9]+ registers|[0-9]+ bytes spill stores" | tr '\n' ' '; echo " [$name]"

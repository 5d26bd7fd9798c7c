#!/bin/bash
# Build libpsim.so with extra nvcc defines into build/ab/<name>/ for A/B runs
# (select it with PSIM_LIB=build/ab/<name>/libpsim.so). Experiment tooling.
# Usage: tools/build_variant.sh <name> -DPSIM_F32_VAR=0 [...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build/ab/$name; rm -rf $out; mkdir -p $out/obj
ls paper_1705_08210_b200/csrc/*.cu | xargs -P 8 -I{} sh -c \
  'nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
     -Iinclude -Ipaper_1705_08210_b200/csrc '"$*"' -c {} -o '"$out"'/obj/$(basename {} .cu).o'
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libpsim.so $out/obj/*.o
echo $out/libpsim.so

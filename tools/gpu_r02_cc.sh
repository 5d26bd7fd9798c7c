#!/bin/bash
# round 2, call CC: FP32 2-way tile / inner-op A/B at cfg3's n_f (n_v = 100000), product vs
# tools/build_variant.sh builds (PSIM_LIB)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02cc; mkdir -p $O
B="python bench.py --config cfg3 --n-v 100000 --steps 2 --warmup 1 --no-cpu --no-e2e --no-parity"
for r in 1 2; do
  timeout 600 $B > $O/prod_$r.json 2> $O/prod_$r.err
  for v in f32_fadd2 f32_s4 f32_imnmx f32_8x8; do
    PSIM_LIB=build/ab/$v/libpsim.so timeout 600 $B > $O/${v}_$r.json 2> $O/${v}_$r.err
  done
done

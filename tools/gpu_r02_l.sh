#!/bin/bash
# round 2, call L: ncu --set full of the TMA kernels (cfg2 FP64 2-way, FP32 2-way, 3-way single-pivot)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02l; mkdir -p $O
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_minplus2" -s 0 -c 1 -o $O/cfg2_tma python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_cfg2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_minplus2" -s 0 -c 1 -o $O/f32_tma python bench.py --config cfg3 --n-v 16384 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_f32.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_czek3" -s 0 -c 1 -o $O/czek3_single python bench.py --config cfg4 --n-v 1536 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_3.log 2>&1

#!/bin/bash
# round 2, call M: 3-way pivot-transform distance A/B (D=1 vs D=2), parity suite
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02m; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
B="python bench.py --config cfg4 --no-cpu --no-e2e --no-parity --steps 1 --warmup 1"
timeout 900 $B > $O/cfg4_d2.json 2>&1
PSIM_LIB=build/ab/d1/libpsim.so timeout 900 $B > $O/cfg4_d1.json 2>&1
timeout 600 $B --n-v 3000 > $O/n3000_d2.json 2>&1
PSIM_LIB=build/ab/d1/libpsim.so timeout 600 $B --n-v 3000 > $O/n3000_d1.json 2>&1

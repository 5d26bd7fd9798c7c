#!/bin/bash
# round 2, call K: runtime tests after the ring fix; 3-way TMA unroll A/B; ncu of the 3-way TMA box kernel
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02k; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "runtime or pageable or streamed or flattened or golden_case" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="python bench.py --config cfg4 --n-v 3000 --no-cpu --no-e2e --no-parity --steps 2 --warmup 1"
timeout 600 $B > $O/ab3_rolled.json 2>&1
PSIM_LIB=build/ab/kku_2/libpsim.so timeout 600 $B > $O/ab3_kku2.json 2>&1
PSIM_LIB=build/ab/kku_full/libpsim.so timeout 600 $B > $O/ab3_full.json 2>&1
PSIM_NO_TMA=1 timeout 600 $B > $O/ab3_cpasync.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_czek3" -s 1 -c 1 -o $O/czek3_tma python bench.py --config cfg4 --n-v 1536 --no-cpu --no-e2e --no-parity --steps 1 --warmup 1 > $O/ncu3.log 2>&1

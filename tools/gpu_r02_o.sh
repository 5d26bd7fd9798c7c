#!/bin/bash
# round 2, call O: 3-way single-pivot TMA variants (tools/exp_pivot_tma.cu) + source-level ncu of k_czek3
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02o; mkdir -p $O
timeout 300 build/exp_pivot_tma 8192 10000 > $O/exp_pivot_tma_8192.jsonl 2>&1
timeout 300 build/exp_pivot_tma 4096 20000 > $O/exp_pivot_tma_4096.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_czek3" -s 0 -c 1 -o $O/czek3_single python bench.py --config cfg4 --n-v 1536 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_var" -c 21 -o $O/exp_pivot build/exp_pivot_tma 2048 10000 > $O/ncu_exp.log 2>&1
timeout 600 python bench.py --config cfg4 --n-v 3000 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/cfg4_n3000_parity.json 2> $O/cfg4_n3000_parity.err

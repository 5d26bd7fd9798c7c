#!/bin/bash
# round 2, call Q: 3-way TMA pivot loop, stage count x transform distance (tools/exp_pivot_tma.cu)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02q; mkdir -p $O
timeout 300 build/exp_pivot_tma 8192 10000 > $O/exp_pivot_tma_8192.jsonl 2>&1
timeout 300 build/exp_pivot_tma 4096 20000 > $O/exp_pivot_tma_4096.jsonl 2>&1
timeout 300 build/exp_pivot_tma 6144 10000 > $O/exp_pivot_tma_6144.jsonl 2>&1

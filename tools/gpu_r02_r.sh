#!/bin/bash
# round 2, call R: production 3-way TMA loop knobs (transform distance D, pivot box, proxy fence)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02r; mkdir -p $O
timeout 300 build/exp_pivot_tma 8192 10000 16257 > $O/exp_pivot_tma_8192.jsonl 2>&1
timeout 300 build/exp_pivot_tma 4096 20000 16257 > $O/exp_pivot_tma_4096.jsonl 2>&1

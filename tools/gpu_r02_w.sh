#!/bin/bash
# round 2, call W: w16 thread mapping (no duplicate pivot rewrite) vs the 16 x 16 grid
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02w; mkdir -p $O
timeout 300 build/exp_pivot_tma 8192 10000 802819 > $O/exp_pivot_tma_8192.jsonl 2>&1
timeout 300 build/exp_pivot_tma 4096 20000 802819 > $O/exp_pivot_tma_4096.jsonl 2>&1

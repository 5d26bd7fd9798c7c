#!/bin/bash
# round 2, call S: interleaved per-warp pivot transform (tools/exp_pivot_tma.cu variants 14-17)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02s; mkdir -p $O
timeout 300 build/exp_pivot_tma 8192 10000 245891 > $O/exp_pivot_tma_8192.jsonl 2>&1
timeout 300 build/exp_pivot_tma 4096 20000 245891 > $O/exp_pivot_tma_4096.jsonl 2>&1

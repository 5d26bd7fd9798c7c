#!/bin/bash
# round 2, call D: TMA vs cp.async A/B (FP64 tile pipeline)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02d; mkdir -p $O
timeout 300 build/exp_tma 8192 20000 > $O/tma_ab.jsonl 2>&1
timeout 300 build/exp_tma 4096 20000 >> $O/tma_ab.jsonl 2>&1

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02g; mkdir -p $O
timeout 300 build/exp_tma 8192 20000 > $O/tma_pad.jsonl 2>&1

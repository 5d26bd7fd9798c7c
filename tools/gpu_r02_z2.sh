#!/bin/bash
# round 2, call Z2 (2 GPUs): cfg4 N=2 sampled parity from the runtime's scratch box
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02z2; mkdir -p $O
timeout 900 python bench.py --gpus 2 --config cfg4 --n-v 3000 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/cfg4_n3000_n2.json 2> $O/cfg4_n3000_n2.err

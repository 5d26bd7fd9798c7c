#!/bin/bash
# round 2, call E: ncu of the TMA kernel of the A/B (stall reasons, pipes)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02e; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tma" -c 1 -o $O/tma_only build/exp_tma 4096 20000 > $O/ncu2.log 2>&1

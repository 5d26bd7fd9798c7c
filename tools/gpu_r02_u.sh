#!/bin/bash
# round 2, call U: 3-way box kernel with and without the Eq. 1 epilogue (tools/exp_box3.py)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02u; mkdir -p $O
timeout 600 python tools/exp_box3.py 10000 > $O/exp_box3.jsonl 2> $O/exp_box3.err

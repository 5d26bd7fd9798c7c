#!/bin/bash
# 32-row edge tiles for ragged row tiles: GPU suite, one-GPU circulant A/B, default bench.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > $O/pytest_edge.log 2>&1; echo pytest=$? >> $O/pytest_edge.log
tail -3 $O/pytest_edge.log
timeout 600 python tools/exp_local_grids.py > $O/local_grids_edge.jsonl 2>&1
PSIM_NO_EDGE=1 timeout 600 python tools/exp_local_grids.py > $O/local_grids_noedge.jsonl 2>&1
cat $O/local_grids_edge.jsonl $O/local_grids_noedge.jsonl
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > $O/bench_edge.json 2> $O/bench_edge.log
head -c 300 $O/bench_edge.json

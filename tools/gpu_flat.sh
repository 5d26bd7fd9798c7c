#!/bin/bash
# Flattened off-diagonal tasks (kCzek2Flat): GPU suite, then the one-GPU circulant A/B.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > $O/pytest_flat.log 2>&1; echo pytest=$? >> $O/pytest_flat.log
tail -3 $O/pytest_flat.log
timeout 600 python tools/exp_local_grids.py > $O/local_grids_flat.jsonl 2>&1
PSIM_NO_FLAT=1 timeout 600 python tools/exp_local_grids.py > $O/local_grids_noflat.jsonl 2>&1
cat $O/local_grids_flat.jsonl $O/local_grids_noflat.jsonl

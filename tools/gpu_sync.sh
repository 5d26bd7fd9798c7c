#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
for m in 0 1 2 3; do timeout 300 build/exp_sync 8 $m >> $O/exp_sync.jsonl 2>&1; done
echo done

#!/bin/bash
# micro-step loop unroll sweep (exp_minplus built with -DPSIM_KK_UNROLL=1,2,4,8)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
for r in 1 2; do for u in 1 2 4 8; do timeout 300 build/exp_minplus_u$u 8192 20000 >> $O/unroll_sweep.jsonl 2>&1; done; done
echo done

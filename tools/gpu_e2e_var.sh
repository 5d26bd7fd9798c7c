#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
HV=1 NOCLK=1 REPS=8 MODES=1 timeout 600 python tools/exp_e2e.py > $O/exp_e2e_noclk.jsonl 2> $O/exp_e2e_noclk.err
HV=1 NOCLK=1 NOGC=1 REPS=8 MODES=1 timeout 600 python tools/exp_e2e.py > $O/exp_e2e_nogc.jsonl 2> $O/exp_e2e_nogc.err
for r in 1 2; do for u in 1 2 4 8; do timeout 300 build/exp_minplus_u$u 8192 20000 >> $O/unroll_sweep.jsonl 2>&1; done; done
echo done

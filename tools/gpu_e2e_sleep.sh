#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
PSIM_POLL=2 HV=1 NOCLK=1 REPS=10 MODES=1 timeout 600 python tools/exp_e2e.py > $O/exp_e2e_sleep.jsonl 2> $O/exp_e2e_sleep.err
echo done

#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
PSIM_POLL=3 HV=1 NOCLK=1 REPS=10 MODES=1 timeout 600 python tools/exp_e2e.py > $O/exp_e2e_spin3.jsonl 2> $O/exp_e2e_spin3.err
PSIM_POLL=0 HV=1 NOCLK=1 REPS=6 MODES=1 timeout 600 python tools/exp_e2e.py > $O/exp_e2e_spin0.jsonl 2> $O/exp_e2e_spin0.err
echo done

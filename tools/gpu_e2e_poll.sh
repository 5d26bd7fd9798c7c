#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
(cat /proc/meminfo | head -5; cat /proc/loadavg; cat /sys/kernel/mm/transparent_hugepage/enabled; nproc; top -bn1 | head -15) > $O/host_state.txt 2>&1
REPS=8 MODES=1 timeout 800 python tools/exp_e2e.py > $O/exp_e2e_block.jsonl 2> $O/exp_e2e_block.err
PSIM_POLL=1 REPS=8 MODES=1 timeout 800 python tools/exp_e2e.py > $O/exp_e2e_poll.jsonl 2> $O/exp_e2e_poll.err
(cat /proc/loadavg; top -bn1 | head -15) >> $O/host_state.txt 2>&1
echo done

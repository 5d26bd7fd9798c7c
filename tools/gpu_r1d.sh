#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
NOCLK=1 REPS=6 MODES=1 timeout 600 python tools/exp_e2e.py > $O/exp_e2e_final.jsonl 2> $O/exp_e2e_final.err
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.log
echo done

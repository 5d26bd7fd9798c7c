#!/bin/bash
# Full GPU suite, cfg2 e2e breakdown (exp_e2e), cfg4 1-GPU bench line with the pivot-ahead loop.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
REPS=3 MODES=1 timeout 600 python tools/exp_e2e.py > $O/exp_e2e.jsonl 2> $O/exp_e2e.err
timeout 900 python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu > $O/scale_cfg4_n1.json 2> $O/scale_cfg4_n1.log
echo done

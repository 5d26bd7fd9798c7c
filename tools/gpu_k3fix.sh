#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
python -m paper_1705_08210_b200.build > $O/build.log 2>&1
python tools/exp_box3.py 10000 > $O/k3fix_box.jsonl 2>&1
python tools/prof_driver.py czek2 --precision double --n-v 16384 --n-f 20000 --reps 2 > $O/k3fix_k2.jsonl 2>&1
python tools/prof_driver.py czek2 --precision single --n-v 32768 --n-f 20000 --reps 2 >> $O/k3fix_k2.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "3way or czek3 or box or band or golden or output" > $O/pytest_k3fix.log 2>&1; echo rc=$? >> $O/pytest_k3fix.log
echo done

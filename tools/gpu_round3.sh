#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
python -m paper_1705_08210_b200.build > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
timeout 900 python bench.py --config cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu > $O/scale_cfg4_n1.json 2> $O/scale_cfg4_n1.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.log
python tools/prof_driver.py czek3 --precision double --n-v 768 --n-f 10000 --reps 1 > $O/k3_small.jsonl 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_czek3 -c 1 -o $O/prof_k3d_small \
  python tools/prof_driver.py czek3 --precision double --n-v 768 --n-f 10000 --reps 1 > $O/ncu_k3.log 2>&1
echo done

#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
python -m paper_1705_08210_b200.build > $O/build.log 2>&1
timeout 900 python bench.py > $O/bench_cfg2_b.json 2> $O/bench_cfg2_b.log
timeout 900 python bench.py --config cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu > $O/bench_cfg4_b.json 2> $O/bench_cfg4_b.log
echo done

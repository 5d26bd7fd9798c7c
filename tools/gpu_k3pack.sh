#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
python -m paper_1705_08210_b200.build > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_k3pack.log 2>&1; echo rc=$? >> $O/pytest_k3pack.log
python tools/exp_box3.py 10000 > $O/k3pack_box.jsonl 2>&1
timeout 900 python bench.py --config cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu > $O/bench_cfg4_pack.json 2> $O/bench_cfg4_pack.log
echo done

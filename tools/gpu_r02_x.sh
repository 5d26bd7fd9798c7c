#!/bin/bash
# round 2, call X: full GPU suite, cfg2 + cfg4 bench lines, cfg4 launch list (ncu, per-launch times)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02x; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg4.csv python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_cfg4.log 2>&1

#!/bin/bash
# round 2, call I: TMA in the 3-way single-pivot tiles: parity, cfg4 A/B, full cfg2 line
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02i; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 1200 python bench.py --config cfg4 --no-cpu --steps 2 --warmup 3 > $O/bench_cfg4_tma.json 2> $O/bench_cfg4_tma.err
PSIM_NO_TMA=1 timeout 900 python bench.py --config cfg4 --no-cpu --no-e2e --no-parity --steps 1 --warmup 1 > $O/bench_cfg4_cpasync.json 2> $O/bench_cfg4_cpasync.err
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err

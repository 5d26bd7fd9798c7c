#!/bin/bash
# round 2, call H: TMA staging in the production 2-way kernels: parity, then A/B
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02h; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --no-cpu --no-e2e > $O/bench_cfg2_tma.json 2> $O/bench_cfg2_tma.err
PSIM_NO_TMA=1 timeout 900 python bench.py --no-cpu --no-e2e --no-parity > $O/bench_cfg2_cpasync.json 2> $O/bench_cfg2_cpasync.err
timeout 900 python bench.py --config cfg3 --no-cpu --no-e2e --steps 2 > $O/bench_cfg3_tma.json 2> $O/bench_cfg3_tma.err
PSIM_NO_TMA=1 timeout 900 python bench.py --config cfg3 --no-cpu --no-e2e --no-parity --steps 2 > $O/bench_cfg3_cpasync.json 2> $O/bench_cfg3_cpasync.err

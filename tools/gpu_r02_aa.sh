#!/bin/bash
# round 2, call AA (4 GPUs): 2-way circulant with the off-diagonal tasks on a second compute stream
# (no drain between the diagonal grid and the rest): NCCL / runtime tests, cfg2 N=2/4, cfg3 N=4
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02aa; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_nccl.py -x -q -p no:cacheprovider > $O/pytest_rt.log 2>&1; echo "rc=$?" >> $O/pytest_rt.log
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu > $O/bench_cfg2_n2.json 2> $O/bench_cfg2_n2.err
timeout 900 python bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu > $O/bench_cfg2_n4.json 2> $O/bench_cfg2_n4.err
timeout 1200 python bench.py --gpus 4 --config cfg3 --steps 2 --warmup 3 --no-cpu > $O/bench_cfg3_n4.json 2> $O/bench_cfg3_n4.err

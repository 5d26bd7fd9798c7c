#!/bin/bash
# round 2, call Y (4 GPUs): GPU suite incl. NCCL world 2/4, cfg2 / cfg4 at N = 2 / 4 (bench self-launch),
# cfg4 n_v=3000 launch list on one GPU (share of the two-pivot packed grid)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02y; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench_cfg2_n2.json 2> $O/bench_cfg2_n2.err
timeout 900 python bench.py --gpus 4 --steps 5 --warmup 3 > $O/bench_cfg2_n4.json 2> $O/bench_cfg2_n4.err
timeout 900 python bench.py --gpus 2 --config cfg4 --steps 2 --warmup 3 > $O/bench_cfg4_n2.json 2> $O/bench_cfg4_n2.err
timeout 900 python bench.py --gpus 4 --config cfg4 --steps 2 --warmup 3 > $O/bench_cfg4_n4.json 2> $O/bench_cfg4_n4.err
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg4_n3000.csv python bench.py --config cfg4 --n-v 3000 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_cfg4_n3000.log 2>&1

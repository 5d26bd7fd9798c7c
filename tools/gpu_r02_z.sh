#!/bin/bash
# round 2, call Z (2 GPUs): runtime / NCCL tests after the psim_out_t scratch fields, cfg4 N=2 sampled
# parity from the runtime's scratch box, cfg1 small-problem latency (tools/exp_small.py, bench --config cfg1)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02z; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_nccl.py -x -q -p no:cacheprovider > $O/pytest_rt.log 2>&1; echo "rc=$?" >> $O/pytest_rt.log
timeout 900 python bench.py --gpus 2 --config cfg4 --n-v 3000 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/cfg4_n3000_n2.json 2> $O/cfg4_n3000_n2.err
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/exp_small.py > $O/exp_small.jsonl 2> $O/exp_small.err
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/exp_small.py 1000 2000 >> $O/exp_small.jsonl 2>> $O/exp_small.err
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config cfg1 --steps 20 --warmup 5 > $O/bench_cfg1.json 2> $O/bench_cfg1.err

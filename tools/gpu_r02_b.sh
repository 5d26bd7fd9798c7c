#!/bin/bash
# round 2, call B: the C++ runtime on 2 GPUs (ctypes-only tests, NCCL parity via
# run_2way/run_3way transport="nccl"), then bench N=2 through RuntimeBench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/r02b
timeout 900 python -m pytest tests/test_gpu_runtime.py -x -q -p no:cacheprovider > gpurun_out/r02b/pytest_runtime.log 2>&1
echo "rc=$?" >> gpurun_out/r02b/pytest_runtime.log
timeout 1200 python -m pytest tests/test_gpu_nccl.py -x -q -p no:cacheprovider > gpurun_out/r02b/pytest_nccl.log 2>&1
echo "rc=$?" >> gpurun_out/r02b/pytest_nccl.log
timeout 900 python bench.py --gpus 2 --no-cpu > gpurun_out/r02b/bench_n2.json 2> gpurun_out/r02b/bench_n2.err; echo "rc=$?" >> gpurun_out/r02b/bench_n2.err
timeout 900 python bench.py --gpus 2 --config cfg4 --no-cpu > gpurun_out/r02b/bench_cfg4_n2.json 2> gpurun_out/r02b/bench_cfg4_n2.err; echo "rc=$?" >> gpurun_out/r02b/bench_cfg4_n2.err

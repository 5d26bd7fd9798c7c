#!/bin/bash
# round 2, call J: 4 GPUs -- NCCL parity at world 4 (runtime), scaling lines cfg2..cfg5
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02j; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_runtime.py -x -q -p no:cacheprovider > $O/pytest_mgpu.log 2>&1; echo "rc=$?" >> $O/pytest_mgpu.log
for c in cfg2 cfg3 cfg4; do
  timeout 1200 python bench.py --gpus 4 --config $c --no-cpu > $O/bench_${c}_n4.json 2> $O/bench_${c}_n4.err
done
timeout 1200 python bench.py --gpus 4 --config cfg5 --no-cpu --no-e2e > $O/bench_cfg5_n4.json 2> $O/bench_cfg5_n4.err
for c in cfg2 cfg3; do
  timeout 1200 python bench.py --gpus 2 --config $c --no-cpu > $O/bench_${c}_n2.json 2> $O/bench_${c}_n2.err
done

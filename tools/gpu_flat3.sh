#!/bin/bash
# 3-way flattened-box check: GPU tests, then cfg4 at N = 2 and 4 (torchrun).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 \
  bench.py --gpus 2 --config cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu > $O/scale_cfg4_n2.json 2> $O/scale_cfg4_n2.log
timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 \
  bench.py --gpus 4 --config cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu > $O/scale_cfg4_n4.json 2> $O/scale_cfg4_n4.log
echo done

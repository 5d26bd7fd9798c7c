#!/bin/bash
# f1 check: full GPU test suite on GPU 0, then the NCCL parity + output check on all GPUs.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
N=${1:-2}
python -m paper_1705_08210_b200.build > $O/build.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
timeout 900 torchrun --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  tools/mgpu_check.py > $O/mgpu_check_$N.jsonl 2> $O/mgpu_check_$N.err; echo rc=$? >> $O/mgpu_check_$N.err
echo done

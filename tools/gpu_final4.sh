#!/bin/bash
# Final 4-GPU pass: GPU suite, NCCL parity at 2 and 4, cfg2 at N = 2, 4 (contract K/W, e2e).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
for n in 2 4; do
  timeout 600 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + n)) \
    tools/mgpu_check.py > $O/mgpu_check_$n.jsonl 2> $O/mgpu_check_$n.err; echo rc=$? >> $O/mgpu_check_$n.err
  timeout 900 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29610 + n)) \
    bench.py --gpus $n --steps 3 --warmup 3 --no-cpu > $O/scale_cfg2_n$n.json 2> $O/scale_cfg2_n$n.log
done
echo done

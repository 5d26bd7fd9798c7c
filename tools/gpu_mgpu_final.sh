#!/bin/bash
# 2/4-GPU refresh: NCCL parity check, cfg2 (contract K/W) and cfg4 at N = 2, 4 with e2e.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
timeout 600 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
  tools/mgpu_check.py > $O/mgpu_check_2.jsonl 2> $O/mgpu_check_2.err; echo rc=$? >> $O/mgpu_check_2.err
for n in 2 4; do
  timeout 900 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29540 + n)) \
    bench.py --gpus $n --steps 3 --warmup 3 --no-cpu > $O/scale_cfg2_n$n.json 2> $O/scale_cfg2_n$n.log
  timeout 1200 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29550 + n)) \
    bench.py --gpus $n --config cfg4 --steps 1 --warmup 1 --no-cpu > $O/scale_cfg4_n$n.json 2> $O/scale_cfg4_n$n.log
done
echo done

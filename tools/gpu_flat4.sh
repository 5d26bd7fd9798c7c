#!/bin/bash
# 4-GPU check of the flattened tasks: NCCL parity (mgpu_check) and cfg2 at N = 2, 4.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 \
  tools/mgpu_check.py > $O/mgpu_check_4.jsonl 2> $O/mgpu_check_4.err; echo rc=$? >> $O/mgpu_check_4.err
for n in 4 2; do
  timeout 900 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29540 + n)) \
    bench.py --gpus $n --steps 3 --warmup 3 --no-cpu > $O/scale_cfg2_n$n.json 2> $O/scale_cfg2_n$n.log
done
tail -2 $O/mgpu_check_4.err; grep -c '"ok": true' $O/mgpu_check_4.jsonl; wc -l < $O/mgpu_check_4.jsonl
for n in 4 2; do head -c 400 $O/scale_cfg2_n$n.json; echo; done

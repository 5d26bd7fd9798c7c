#!/bin/bash
# cfg3 (2-way FP32 50000 x 200000) at N = 4, 2 with the flattened + edge tasks.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
for n in 4 2; do
  timeout 900 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29560 + n)) \
    bench.py --gpus $n --config cfg3 --steps 1 --warmup 1 --no-cpu > $O/scale_cfg3_n$n.json 2> $O/scale_cfg3_n$n.log
  head -c 300 $O/scale_cfg3_n$n.json; echo
done

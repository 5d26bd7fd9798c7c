#!/bin/bash
# cfg3 at N = 2, 4 and cfg5 at N = 4 with the current library (1 warm-up + 1 timed step).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
for n in 2 4; do
  timeout 1200 torchrun --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29570 + n)) \
    bench.py --gpus $n --config cfg3 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/scale_cfg3_n$n.json 2> $O/scale_cfg3_n$n.log
done
timeout 1200 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29579 \
  bench.py --gpus 4 --config cfg5 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/scale_cfg5_n4.json 2> $O/scale_cfg5_n4.log
echo done

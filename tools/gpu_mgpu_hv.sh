#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
N=${1:-2}
timeout 600 torchrun --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29561 \
  tools/mgpu_check.py > $O/mgpu_check_$N.jsonl 2> $O/mgpu_check_$N.err; echo rc=$? >> $O/mgpu_check_$N.err
timeout 900 torchrun --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29562 \
  bench.py --gpus $N --steps 3 --warmup 3 --no-cpu > $O/scale_cfg2_n$N.json 2> $O/scale_cfg2_n$N.log
echo done

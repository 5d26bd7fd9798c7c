#!/bin/bash
# Multi-GPU bench sweep on one box: configs x N (torchrun), 1 warm-up + 1 timed step each.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
run() {  # config N steps warmup
  local port=$((29600 + RANDOM % 300))
  if [ "$2" = "1" ]; then
    timeout 1200 python bench.py --config $1 --steps $3 --warmup $4 --no-e2e --no-cpu > $O/scale_$1_n$2.json 2> $O/scale_$1_n$2.log
  else
    timeout 1200 torchrun --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $port \
      bench.py --gpus $2 --config $1 --steps $3 --warmup $4 --no-e2e --no-cpu > $O/scale_$1_n$2.json 2> $O/scale_$1_n$2.log
  fi
  echo "$1 n$2 rc=$?" >> $O/scale_status.txt
}
for spec in "$@"; do
  IFS=: read cfg n steps warm <<< "$spec"
  run $cfg $n ${steps:-1} ${warm:-1}
done
echo done

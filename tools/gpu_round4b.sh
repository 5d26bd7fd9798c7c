#!/bin/bash
# 4-GPU session: NCCL parity + output check at 4 and 2 ranks, then the scaling sweep.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
python -m paper_1705_08210_b200.build > $O/build.log 2>&1
timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
  tools/mgpu_check.py > $O/mgpu_check_4.jsonl 2> $O/mgpu_check_4.err; echo rc=$? >> $O/mgpu_check_4.err
timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  tools/mgpu_check.py > $O/mgpu_check_2.jsonl 2> $O/mgpu_check_2.err; echo rc=$? >> $O/mgpu_check_2.err
timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu > $O/bench_cfg2_n4.json 2> $O/bench_cfg2_n4.log
timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 \
  bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu > $O/bench_cfg2_n2.json 2> $O/bench_cfg2_n2.log
bash tools/gpu_scale.sh cfg4:2 cfg4:4 cfg3:4 > /dev/null 2>&1
echo done

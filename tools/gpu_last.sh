#!/bin/bash
# Final tree: GPU suite + smoke on GPU 0, 2-GPU NCCL parity (mgpu_check).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? >> $O/smoke.log
timeout 600 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
  tools/mgpu_check.py > $O/mgpu_check_2.jsonl 2> $O/mgpu_check_2.err; echo rc=$? >> $O/mgpu_check_2.err
tail -2 $O/pytest_gpu.log; tail -1 $O/smoke.log; tail -1 $O/mgpu_check_2.err
grep -c '"ok": true' $O/mgpu_check_2.jsonl; grep -vc '"ok": true' $O/mgpu_check_2.jsonl

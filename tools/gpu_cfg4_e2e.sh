#!/bin/bash
# cfg4 on 1 GPU with the public-API e2e leg (3-way), after a small smoke of the same path.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
timeout 300 python bench.py --config cfg4 --n-v 1200 --steps 1 --warmup 1 --no-cpu > $O/cfg4_small.json 2> $O/cfg4_small.log
timeout 900 python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu > $O/scale_cfg4_n1.json 2> $O/scale_cfg4_n1.log
echo done

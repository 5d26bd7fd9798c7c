#!/bin/bash
# Round-1 final evidence: launch list of the default bench, ncu --set full of the 2-way FP64 and
# FP32 kernels (rolled / x4 micro-step loops), cfg3 1-GPU line.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_minplus2 -c 1 -o $O/prof_k2d_final \
  python tools/prof_driver.py czek2 --precision double --n-v 4096 --reps 1 > $O/ncu_k2d.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_minplus2 -c 1 -o $O/prof_k2s_final \
  python tools/prof_driver.py czek2 --precision single --n-v 4096 --n-f 50000 --reps 1 > $O/ncu_k2s.log 2>&1
timeout 900 python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/scale_cfg3_n1.json 2> $O/scale_cfg3_n1.log
echo done

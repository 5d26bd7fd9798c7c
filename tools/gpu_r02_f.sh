#!/bin/bash
# round 2, call F: TMA unroll variants; the bench launch list; ncu --set full of the
# dominant cfg2 kernel (DRAM traffic per launch for roofline.traffic)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02f; mkdir -p $O
timeout 300 build/exp_tma 8192 20000 > $O/tma_unroll.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > $O/ncu_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_minplus2" -s 3 -c 1 -o $O/cfg2_kernel python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-parity > $O/ncu_full.log 2>&1

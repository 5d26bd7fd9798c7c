#!/bin/bash
# ncu evidence for the bench's dominant kernel at the cfg2 size + the bench launch list.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
python -m paper_1705_08210_b200.build > $O/build.log 2>&1
python tools/prof_driver.py czek2 --precision double --n-v 40000 --n-f 20000 --reps 1 > $O/cfg2_plain.jsonl 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_minplus2 -c 1 \
  -o $O/prof_cfg2 python tools/prof_driver.py czek2 --precision double --n-v 40000 --n-f 20000 --reps 1 > $O/ncu_cfg2.log 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/bench_small.json 2>$O/bench_small.log && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_launches.log 2>&1
python tools/prof_driver.py czek2 --precision single --n-v 16384 --n-f 50000 --reps 1 > /dev/null 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_minplus2 -c 1 \
  -o $O/prof_k2s_v2 python tools/prof_driver.py czek2 --precision single --n-v 16384 --n-f 50000 --reps 1 > $O/ncu_k2s.log 2>&1
echo done

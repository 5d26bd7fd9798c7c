#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
python -m paper_1705_08210_b200.build > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
python tools/prof_driver.py czek2 --precision double --n-v 16384 --n-f 20000 --reps 2 > $O/r2_k2.jsonl 2>&1
python tools/prof_driver.py czek2 --precision single --n-v 16384 --n-f 50000 --reps 2 >> $O/r2_k2.jsonl 2>&1
python tools/prof_driver.py czek2 --precision double --n-v 40000 --n-f 20000 --reps 1 >> $O/r2_k2.jsonl 2>&1 && \
timeout 900 ncu --metrics $M --replay-mode application --clock-control none -k regex:k_minplus2 -c 1 --csv \
  python tools/prof_driver.py czek2 --precision double --n-v 40000 --n-f 20000 --reps 1 > $O/traffic_cfg2_r2.csv 2>&1
timeout 900 python bench.py --config cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu > $O/bench_cfg4_r2.json 2> $O/bench_cfg4_r2.log
echo done

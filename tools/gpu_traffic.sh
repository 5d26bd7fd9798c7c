#!/bin/bash
# DRAM traffic of the dominant kernels at bench size (application replay, few metrics)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct
python tools/prof_driver.py czek2 --precision double --n-v 40000 --n-f 20000 --reps 1 > $O/t_cfg2_plain.jsonl 2>&1 && \
timeout 900 ncu --metrics $M --replay-mode application --clock-control none -k regex:k_minplus2 -c 1 --csv \
  python tools/prof_driver.py czek2 --precision double --n-v 40000 --n-f 20000 --reps 1 > $O/traffic_cfg2.csv 2>&1
python tools/prof_driver.py czek3 --precision double --n-v 3000 --n-f 10000 --reps 1 > $O/t_k3_plain.jsonl 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_czek3 -c 1 -o $O/prof_k3d \
  python tools/prof_driver.py czek3 --precision double --n-v 3000 --n-f 10000 --reps 1 > $O/ncu_k3.log 2>&1
echo done

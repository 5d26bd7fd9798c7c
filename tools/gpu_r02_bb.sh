#!/bin/bash
# round 2, call BB: DRAM bytes per launch of the dominant kernel at the cfg4 and cfg3 bench configs
# (ncu dram metrics only: one replay pass), for roofline.traffic
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02bb; mkdir -p $O
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 1200 ncu --metrics $M --clock-control none -k regex:"k_czek3" -c 16 --csv --log-file $O/traffic_cfg4.csv python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_cfg4.log 2>&1
timeout 1200 ncu --metrics $M --clock-control none -k regex:"k_minplus2" -c 2 --csv --log-file $O/traffic_cfg3.csv python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_cfg3.log 2>&1

#!/bin/bash
# Round-end evidence after the flattened / edge tasks: GPU suite, smoke, default bench, reference
# arm, launch list of the default bench, ncu --set full of the 32-row edge grid.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
bash tools/gpu_final.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_launch.log 2>&1
# second k_minplus2 launch of a 4104-vector single-slab task = its edge grid (8 rows)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_minplus2 --launch-skip 1 -c 1 \
  -o $O/prof_edge python tools/prof_driver.py czek2 --precision double --n-v 4104 --reps 1 > $O/ncu_edge.log 2>&1
echo done2

#!/bin/bash
# 3-way box layouts: per-layout rates (exp_box3), then ncu --set full of the
# single-pivot and two-segment grids of a FLAT_COLS face box.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
python tools/exp_box3.py 10000 > $O/box3_layouts.jsonl 2> $O/box3_layouts.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_czek3 -c 2 \
  -o $O/prof_flat3 python tools/exp_box3.py 10000 "face small" > $O/ncu_flat3.log 2>&1
echo done

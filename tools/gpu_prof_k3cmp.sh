#!/bin/bash
# ncu --set full of the pivot mainloop experiment (exp_pivot v1) vs the product
# 3-way kernel on an all-full-tile volume box, to locate the product's ~5% gap.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
python -m paper_1705_08210_b200.build > $O/build.log 2>&1
build/exp_pivot 4096 10000 > $O/k3cmp_exp.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base mangled \
  -k regex:Li1EEvPKd -c 1 -o $O/prof_exp_v1 build/exp_pivot 4096 10000 > $O/ncu_exp.log 2>&1
python tools/exp_box3.py 10000 "512^3" > $O/k3cmp_box.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_czek3 -c 1 \
  -o $O/prof_box512 python tools/exp_box3.py 10000 "512^3" > $O/ncu_box.log 2>&1
echo done

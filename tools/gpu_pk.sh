#!/bin/bash
# 3-way pivot-loop unroll A/B (build/libpsim_pk{2,4}.so vs the product library, full unroll)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
for r in 1 2; do
for lib in cur pk2 pk4; do
  if [ $lib = cur ]; then unset PSIM_LIB; else export PSIM_LIB=build/libpsim_$lib.so; fi
  timeout 300 python tools/exp_box3.py 10000 "volume 1024" | sed "s/^/$lib /" >> $O/pk_ab.txt 2>> $O/pk_ab.err
  timeout 300 python tools/exp_box3.py 10000 "diag pivots [2000" | sed "s/^/$lib /" >> $O/pk_ab.txt 2>> $O/pk_ab.err
done
done
echo done

#!/bin/bash
# unroll change A/B: old library (build/libpsim_old.so) vs new, 2-way FP64/FP32 and 3-way boxes
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
for lib in old new; do
  if [ $lib = old ]; then export PSIM_LIB=build/libpsim_old.so; else unset PSIM_LIB; fi
  timeout 300 python tools/prof_driver.py czek2 --precision double --n-v 16384 --n-f 20000 --reps 3 > $O/ua_${lib}_f64.jsonl 2>&1
  timeout 300 python tools/prof_driver.py czek2 --precision single --n-v 24576 --n-f 50000 --reps 3 > $O/ua_${lib}_f32.jsonl 2>&1
  timeout 600 python tools/exp_box3.py 10000 "volume 1024" > $O/ua_${lib}_box.jsonl 2>&1
done
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
echo done

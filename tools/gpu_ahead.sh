#!/bin/bash
# GPU suite (new plug-point tests included), host copy probe, and the 3-way
# pivot-ahead A/B (build/libpsim_old.so = two barriers per stage).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
nvidia-smi topo -m > $O/topo.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
timeout 300 python tools/exp_h2d.py 4 > $O/h2d.json 2> $O/h2d.err
for lib in old new; do
  if [ $lib = old ]; then export PSIM_LIB=build/libpsim_old.so; else unset PSIM_LIB; fi
  timeout 600 python tools/exp_box3.py 10000 "volume 1024" > $O/ab_$lib.jsonl 2>> $O/ab.err
  timeout 600 python tools/exp_box3.py 10000 "face I<J=K" >> $O/ab_$lib.jsonl 2>> $O/ab.err
  timeout 600 python tools/exp_box3.py 10000 "diag pivots [2000" >> $O/ab_$lib.jsonl 2>> $O/ab.err
done
echo done

#!/bin/bash
# GPU session: peaks, kernel timings, ncu captures of the 2-way kernel, tests, bench.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
python -m paper_1705_08210_b200.build > $O/build.log 2>&1
for v in 0 2; do python tools/prof_driver.py peak --precision double --variant $v --reps 2 >> $O/peak.jsonl; done
for v in 0 1 2; do python tools/prof_driver.py peak --precision single --variant $v --reps 2 >> $O/peak.jsonl; done
python tools/prof_driver.py czek2 --precision double --n-v 8192 --reps 3 >> $O/k2.jsonl 2>>$O/k2.err
python tools/prof_driver.py czek2 --precision single --n-v 16384 --n-f 50000 --reps 3 >> $O/k2.jsonl 2>>$O/k2.err
python tools/prof_driver.py czek3 --precision double --n-v 1536 --n-f 10000 --reps 2 >> $O/k3.jsonl 2>>$O/k3.err
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > $O/bench.json 2> $O/bench.log; echo bench=$? >> $O/bench.log
python tools/prof_driver.py czek2 --precision double --n-v 4096 --reps 1 > /dev/null && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_minplus2 -c 1 -o $O/prof_k2d \
  python tools/prof_driver.py czek2 --precision double --n-v 4096 --reps 1 > $O/ncu_k2d.log 2>&1
python tools/prof_driver.py czek2 --precision single --n-v 4096 --n-f 50000 --reps 1 > /dev/null && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_minplus2 -c 1 -o $O/prof_k2s \
  python tools/prof_driver.py czek2 --precision single --n-v 4096 --n-f 50000 --reps 1 > $O/ncu_k2s.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_peak -s 1 -c 1 -o $O/prof_peakd \
  python tools/prof_driver.py peak --precision double --variant 0 --reps 1 > $O/ncu_peak.log 2>&1
echo done

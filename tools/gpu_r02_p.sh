#!/bin/bash
# round 2, call P: 3-way single-pivot TMA variants (tools/exp_pivot_tma.cu), ncu per variant
# (summarised on the box; reports kept only while gpurun_out stays small)
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02p; mkdir -p $O
timeout 300 build/exp_pivot_tma 8192 10000 > $O/exp_pivot_tma_8192.jsonl 2>&1
timeout 300 build/exp_pivot_tma 4096 20000 > $O/exp_pivot_tma_4096.jsonl 2>&1
for v in 0 1 2 3 4; do
  m=$((1 << v))
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_var" -c 1 -o $O/var$v build/exp_pivot_tma 2048 10000 $m > $O/ncu_var$v.log 2>&1
  python tools/ncu_summary.py $O/var$v.ncu-rep "exp_pivot_tma variant $v" > $O/ncu_var$v.md 2>&1
  ncu -i $O/var$v.ncu-rep --page source --csv --print-source sass > $O/var${v}_src.csv 2>/dev/null
  python tools/ncu_stalls.py $O/var${v}_src.csv > $O/var${v}_stalls.txt 2>&1
  gzip -f $O/var${v}_src.csv
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_czek3" -s 0 -c 1 -o $O/czek3_single python bench.py --config cfg4 --n-v 1536 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_3.log 2>&1
python tools/ncu_summary.py $O/czek3_single.ncu-rep "k_czek3 single-pivot, cfg4 n_v=1536" > $O/ncu_czek3.md 2>&1
ncu -i $O/czek3_single.ncu-rep --page source --csv --print-source sass > $O/czek3_src.csv 2>/dev/null
python tools/ncu_stalls.py $O/czek3_src.csv > $O/czek3_stalls.txt 2>&1
gzip -f $O/czek3_src.csv
timeout 600 python bench.py --config cfg4 --n-v 3000 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/cfg4_n3000_parity.json 2> $O/cfg4_n3000_parity.err
# keep the copy-back under 64 MiB: drop reports if too big
du -sm $O; if [ $(du -sm $O | cut -f1) -gt 55 ]; then rm -f $O/*.ncu-rep; fi

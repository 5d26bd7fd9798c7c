#!/bin/bash
# round 2, call T: 3-way single-pivot tiles on the interleaved per-warp pivot loop
# (minplus_tile_pivot_ilv): GPU suite, cfg4 bench, ncu summary of k_czek3
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02t; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu > $O/bench_cfg4.json 2> $O/bench_cfg4.err
timeout 600 python bench.py --config cfg4 --n-v 3000 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/cfg4_n3000.json 2> $O/cfg4_n3000.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_czek3" -s 0 -c 1 -o $O/czek3_single python bench.py --config cfg4 --n-v 1536 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_3.log 2>&1
python tools/ncu_summary.py $O/czek3_single.ncu-rep "k_czek3 single-pivot (interleaved pivot loop), cfg4 n_v=1536" > $O/ncu_czek3.md 2>&1
ncu -i $O/czek3_single.ncu-rep --page source --csv --print-source sass > $O/czek3_src.csv 2>/dev/null
python tools/ncu_stalls.py $O/czek3_src.csv > $O/czek3_stalls.txt 2>&1
gzip -f $O/czek3_src.csv
du -sm $O; if [ $(du -sm $O | cut -f1) -gt 55 ]; then rm -f $O/*.ncu-rep; fi

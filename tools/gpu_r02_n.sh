#!/bin/bash
# round 2, call N (re-entry): HEAD check — GPU suite, smoke, default bench, reference arm, cfg4 line
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02n; mkdir -p $O
nvidia-smi -L > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err

#!/bin/bash
# round 2, call V: specialised single-pivot 3-way epilogue: box rates with / without the epilogue, 3-way GPU tests
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02v; mkdir -p $O
timeout 300 python tools/exp_box3.py 10000 "volume 1024" > $O/exp_box3.jsonl 2> $O/exp_box3.err
timeout 300 python tools/exp_box3.py 10000 "diag pivots [2000" >> $O/exp_box3.jsonl 2>> $O/exp_box3.err
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "3way or czek3 or box or config_shaped or golden" > $O/pytest_3.log 2>&1; echo "rc=$?" >> $O/pytest_3.log

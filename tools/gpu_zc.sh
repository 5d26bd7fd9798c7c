#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
python -m paper_1705_08210_b200.build > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "band or streamed or output or host" > $O/pytest_zc.log 2>&1; echo rc=$? >> $O/pytest_zc.log
timeout 900 python bench.py --no-cpu > $O/bench_zc_direct.json 2> $O/bench_zc_direct.log
PSIM_HOST_OUTPUT=bands timeout 900 python bench.py --no-cpu > $O/bench_zc_bands.json 2> $O/bench_zc_bands.log
echo done

#!/bin/bash
# Round-end check of the committed tree: GPU suite, smoke(), default bench (contract K/W, CPU baseline).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$? >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.log
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.log
echo done

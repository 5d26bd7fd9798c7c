#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
python -m paper_1705_08210_b200.build > $O/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "streamed or band or output or golden" > $O/pytest_st.log 2>&1; echo rc=$? >> $O/pytest_st.log
timeout 900 python tools/exp_e2e.py > $O/exp_e2e4.jsonl 2>&1
timeout 900 python bench.py --no-cpu > $O/bench_st.json 2> $O/bench_st.log
echo done

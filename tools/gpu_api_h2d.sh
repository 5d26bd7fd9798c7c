#!/bin/bash
# New GPU tests (plug-point module), host placement / copy bandwidth probe.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
O=gpurun_out
timeout 600 python -m pytest tests/test_mingemm_api.py tests/test_capi.py -q > $O/pytest_api.log 2>&1; echo pytest=$? >> $O/pytest_api.log
nvidia-smi topo -m > $O/topo.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
(command -v numactl && numactl -H) > $O/numa.txt 2>&1
timeout 300 python tools/exp_h2d.py 4 > $O/h2d.json 2> $O/h2d.err
echo done

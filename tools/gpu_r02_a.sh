#!/bin/bash
# round 2, call A: full GPU suite at 2 GPUs (incl. NCCL parity), smoke, bench N=1 and N=2
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out/r02a
nvidia-smi -L > gpurun_out/r02a/gpus.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02a/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02a/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02a/smoke.log
timeout 900 python bench.py > gpurun_out/r02a/bench_n1.json 2> gpurun_out/r02a/bench_n1.err; echo "rc=$?" >> gpurun_out/r02a/bench_n1.err
timeout 900 python bench.py --gpus 2 > gpurun_out/r02a/bench_n2.json 2> gpurun_out/r02a/bench_n2.err; echo "rc=$?" >> gpurun_out/r02a/bench_n2.err
timeout 600 python bench.py --impl reference > gpurun_out/r02a/bench_ref.json 2> gpurun_out/r02a/bench_ref.err

#!/bin/bash
# round 2, call C: full GPU suite (2 GPUs), FP64 mix microbenchmarks, peak variants,
# cfg3 at N=2 through the runtime, ncu of the FP32 2-way and 3-way kernels
cd "$GRAFT_REPO_ROOT" || exit 1
O=gpurun_out/r02c; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 build/exp_fp64_mix 20000 > $O/fp64_mix.jsonl 2> $O/fp64_mix.err
timeout 300 python - > $O/peak_variants.jsonl 2>&1 <<'PY'
import ctypes as C, json
import torch
from paper_1705_08210_b200 import _native as N
for code, name in ((N.F64, "f64"), (N.F32, "f32")):
    for var in range(5):
        if code == N.F64 and var == 1: continue
        cps, cpc = C.c_double(), C.c_double()
        N.call("psim_peak_minplus", code, var, 20000 if code == N.F64 else 40000, C.byref(cps), C.byref(cpc), None)
        print(json.dumps({"dtype": name, "variant": var, "cmp_per_s": cps.value, "cmp_per_clk_sm": cpc.value}))
PY
timeout 1200 python bench.py --gpus 2 --config cfg3 --no-cpu --steps 3 > $O/bench_cfg3_n2.json 2> $O/bench_cfg3_n2.err; echo "rc=$?" >> $O/bench_cfg3_n2.err

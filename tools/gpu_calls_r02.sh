#!/bin/bash
# Round-2 GPU calls (the commands behind profiles/r02_*), one case per call:
#   /usr/local/graft/bin/gpurun [--gpus N] -- "bash tools/gpu_calls_r02.sh <call>"
# Calls a-m were the first session of the round; n-cc this session.
cd "$GRAFT_REPO_ROOT" || exit 1
case "$1" in
a)
  # round 2, call A: full GPU suite at 2 GPUs (incl. NCCL parity), smoke, bench N=1 and N=2
  mkdir -p gpurun_out/r02a
  nvidia-smi -L > gpurun_out/r02a/gpus.txt
  timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02a/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/r02a/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02a/smoke.log
  timeout 900 python bench.py > gpurun_out/r02a/bench_n1.json 2> gpurun_out/r02a/bench_n1.err; echo "rc=$?" >> gpurun_out/r02a/bench_n1.err
  timeout 900 python bench.py --gpus 2 > gpurun_out/r02a/bench_n2.json 2> gpurun_out/r02a/bench_n2.err; echo "rc=$?" >> gpurun_out/r02a/bench_n2.err
  timeout 600 python bench.py --impl reference > gpurun_out/r02a/bench_ref.json 2> gpurun_out/r02a/bench_ref.err
  ;;
b)
  # round 2, call B: the C++ runtime on 2 GPUs (ctypes-only tests, NCCL parity via
  # run_2way/run_3way transport="nccl"), then bench N=2 through RuntimeBench
  mkdir -p gpurun_out/r02b
  timeout 900 python -m pytest tests/test_gpu_runtime.py -x -q -p no:cacheprovider > gpurun_out/r02b/pytest_runtime.log 2>&1
  echo "rc=$?" >> gpurun_out/r02b/pytest_runtime.log
  timeout 1200 python -m pytest tests/test_gpu_nccl.py -x -q -p no:cacheprovider > gpurun_out/r02b/pytest_nccl.log 2>&1
  echo "rc=$?" >> gpurun_out/r02b/pytest_nccl.log
  timeout 900 python bench.py --gpus 2 --no-cpu > gpurun_out/r02b/bench_n2.json 2> gpurun_out/r02b/bench_n2.err; echo "rc=$?" >> gpurun_out/r02b/bench_n2.err
  timeout 900 python bench.py --gpus 2 --config cfg4 --no-cpu > gpurun_out/r02b/bench_cfg4_n2.json 2> gpurun_out/r02b/bench_cfg4_n2.err; echo "rc=$?" >> gpurun_out/r02b/bench_cfg4_n2.err
  ;;
c)
  # round 2, call C: full GPU suite (2 GPUs), FP64 mix microbenchmarks, peak variants,
  # cfg3 at N=2 through the runtime, ncu of the FP32 2-way and 3-way kernels
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
  ;;
d)
  # round 2, call D: TMA vs cp.async A/B (FP64 tile pipeline)
  O=gpurun_out/r02d; mkdir -p $O
  timeout 300 build/exp_tma 8192 20000 > $O/tma_ab.jsonl 2>&1
  timeout 300 build/exp_tma 4096 20000 >> $O/tma_ab.jsonl 2>&1
  ;;
e)
  # round 2, call E: ncu of the TMA kernel of the A/B (stall reasons, pipes)
  O=gpurun_out/r02e; mkdir -p $O
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tma" -c 1 -o $O/tma_only build/exp_tma 4096 20000 > $O/ncu2.log 2>&1
  ;;
f)
  # round 2, call F: TMA unroll variants; the bench launch list; ncu --set full of the
  # dominant cfg2 kernel (DRAM traffic per launch for roofline.traffic)
  O=gpurun_out/r02f; mkdir -p $O
  timeout 300 build/exp_tma 8192 20000 > $O/tma_unroll.jsonl 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > $O/ncu_launch.log 2>&1
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_minplus2" -s 3 -c 1 -o $O/cfg2_kernel python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-parity > $O/ncu_full.log 2>&1
  ;;
g)
  O=gpurun_out/r02g; mkdir -p $O
  timeout 300 build/exp_tma 8192 20000 > $O/tma_pad.jsonl 2>&1
  ;;
h)
  # round 2, call H: TMA staging in the production 2-way kernels: parity, then A/B
  O=gpurun_out/r02h; mkdir -p $O
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
  timeout 900 python bench.py --no-cpu --no-e2e > $O/bench_cfg2_tma.json 2> $O/bench_cfg2_tma.err
  PSIM_NO_TMA=1 timeout 900 python bench.py --no-cpu --no-e2e --no-parity > $O/bench_cfg2_cpasync.json 2> $O/bench_cfg2_cpasync.err
  timeout 900 python bench.py --config cfg3 --no-cpu --no-e2e --steps 2 > $O/bench_cfg3_tma.json 2> $O/bench_cfg3_tma.err
  PSIM_NO_TMA=1 timeout 900 python bench.py --config cfg3 --no-cpu --no-e2e --no-parity --steps 2 > $O/bench_cfg3_cpasync.json 2> $O/bench_cfg3_cpasync.err
  ;;
i)
  # round 2, call I: TMA in the 3-way single-pivot tiles: parity, cfg4 A/B, full cfg2 line
  O=gpurun_out/r02i; mkdir -p $O
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
  timeout 1200 python bench.py --config cfg4 --no-cpu --steps 2 --warmup 3 > $O/bench_cfg4_tma.json 2> $O/bench_cfg4_tma.err
  PSIM_NO_TMA=1 timeout 900 python bench.py --config cfg4 --no-cpu --no-e2e --no-parity --steps 1 --warmup 1 > $O/bench_cfg4_cpasync.json 2> $O/bench_cfg4_cpasync.err
  timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
  ;;
j)
  # round 2, call J: 4 GPUs -- NCCL parity at world 4 (runtime), scaling lines cfg2..cfg5
  O=gpurun_out/r02j; mkdir -p $O
  nvidia-smi topo -m > $O/topo.txt 2>&1
  timeout 1500 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_runtime.py -x -q -p no:cacheprovider > $O/pytest_mgpu.log 2>&1; echo "rc=$?" >> $O/pytest_mgpu.log
  for c in cfg2 cfg3 cfg4; do
    timeout 1200 python bench.py --gpus 4 --config $c --no-cpu > $O/bench_${c}_n4.json 2> $O/bench_${c}_n4.err
  done
  timeout 1200 python bench.py --gpus 4 --config cfg5 --no-cpu --no-e2e > $O/bench_cfg5_n4.json 2> $O/bench_cfg5_n4.err
  for c in cfg2 cfg3; do
    timeout 1200 python bench.py --gpus 2 --config $c --no-cpu > $O/bench_${c}_n2.json 2> $O/bench_${c}_n2.err
  done
  ;;
k)
  # round 2, call K: runtime tests after the ring fix; 3-way TMA unroll A/B; ncu of the 3-way TMA box kernel
  O=gpurun_out/r02k; mkdir -p $O
  timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "runtime or pageable or streamed or flattened or golden_case" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
  B="python bench.py --config cfg4 --n-v 3000 --no-cpu --no-e2e --no-parity --steps 2 --warmup 1"
  timeout 600 $B > $O/ab3_rolled.json 2>&1
  PSIM_LIB=build/ab/kku_2/libpsim.so timeout 600 $B > $O/ab3_kku2.json 2>&1
  PSIM_LIB=build/ab/kku_full/libpsim.so timeout 600 $B > $O/ab3_full.json 2>&1
  PSIM_NO_TMA=1 timeout 600 $B > $O/ab3_cpasync.json 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_czek3" -s 1 -c 1 -o $O/czek3_tma python bench.py --config cfg4 --n-v 1536 --no-cpu --no-e2e --no-parity --steps 1 --warmup 1 > $O/ncu3.log 2>&1
  ;;
l)
  # round 2, call L: ncu --set full of the TMA kernels (cfg2 FP64 2-way, FP32 2-way, 3-way single-pivot)
  O=gpurun_out/r02l; mkdir -p $O
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_minplus2" -s 0 -c 1 -o $O/cfg2_tma python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_cfg2.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_minplus2" -s 0 -c 1 -o $O/f32_tma python bench.py --config cfg3 --n-v 16384 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_f32.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_czek3" -s 0 -c 1 -o $O/czek3_single python bench.py --config cfg4 --n-v 1536 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_3.log 2>&1
  ;;
m)
  # round 2, call M: 3-way pivot-transform distance A/B (D=1 vs D=2), parity suite
  O=gpurun_out/r02m; mkdir -p $O
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
  B="python bench.py --config cfg4 --no-cpu --no-e2e --no-parity --steps 1 --warmup 1"
  timeout 900 $B > $O/cfg4_d2.json 2>&1
  PSIM_LIB=build/ab/d1/libpsim.so timeout 900 $B > $O/cfg4_d1.json 2>&1
  timeout 600 $B --n-v 3000 > $O/n3000_d2.json 2>&1
  PSIM_LIB=build/ab/d1/libpsim.so timeout 600 $B --n-v 3000 > $O/n3000_d1.json 2>&1
  ;;
n)
  # round 2, call N (re-entry): HEAD check — GPU suite, smoke, default bench, reference arm, cfg4 line
  O=gpurun_out/r02n; mkdir -p $O
  nvidia-smi -L > $O/smi.txt 2>&1
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
  timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
  timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
  timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
  ;;
o)
  # round 2, call O: 3-way single-pivot TMA variants (tools/exp_pivot_tma.cu) + source-level ncu of k_czek3
  O=gpurun_out/r02o; mkdir -p $O
  timeout 300 build/exp_pivot_tma 8192 10000 > $O/exp_pivot_tma_8192.jsonl 2>&1
  timeout 300 build/exp_pivot_tma 4096 20000 > $O/exp_pivot_tma_4096.jsonl 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_czek3" -s 0 -c 1 -o $O/czek3_single python bench.py --config cfg4 --n-v 1536 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_3.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_var" -c 21 -o $O/exp_pivot build/exp_pivot_tma 2048 10000 > $O/ncu_exp.log 2>&1
  timeout 600 python bench.py --config cfg4 --n-v 3000 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/cfg4_n3000_parity.json 2> $O/cfg4_n3000_parity.err
  ;;
p)
  # round 2, call P: 3-way single-pivot TMA variants (tools/exp_pivot_tma.cu), ncu per variant
  # (summarised on the box; reports kept only while gpurun_out stays small)
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
  ;;
q)
  # round 2, call Q: 3-way TMA pivot loop, stage count x transform distance (tools/exp_pivot_tma.cu)
  O=gpurun_out/r02q; mkdir -p $O
  timeout 300 build/exp_pivot_tma 8192 10000 > $O/exp_pivot_tma_8192.jsonl 2>&1
  timeout 300 build/exp_pivot_tma 4096 20000 > $O/exp_pivot_tma_4096.jsonl 2>&1
  timeout 300 build/exp_pivot_tma 6144 10000 > $O/exp_pivot_tma_6144.jsonl 2>&1
  ;;
r)
  # round 2, call R: production 3-way TMA loop knobs (transform distance D, pivot box, proxy fence)
  O=gpurun_out/r02r; mkdir -p $O
  timeout 300 build/exp_pivot_tma 8192 10000 16257 > $O/exp_pivot_tma_8192.jsonl 2>&1
  timeout 300 build/exp_pivot_tma 4096 20000 16257 > $O/exp_pivot_tma_4096.jsonl 2>&1
  ;;
s)
  # round 2, call S: interleaved per-warp pivot transform (tools/exp_pivot_tma.cu variants 14-17)
  O=gpurun_out/r02s; mkdir -p $O
  timeout 300 build/exp_pivot_tma 8192 10000 245891 > $O/exp_pivot_tma_8192.jsonl 2>&1
  timeout 300 build/exp_pivot_tma 4096 20000 245891 > $O/exp_pivot_tma_4096.jsonl 2>&1
  ;;
t)
  # round 2, call T: 3-way single-pivot tiles on the interleaved per-warp pivot loop
  # (minplus_tile_pivot_ilv): GPU suite, cfg4 bench, ncu summary of k_czek3
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
  ;;
u)
  # round 2, call U: 3-way box kernel with and without the Eq. 1 epilogue (tools/exp_box3.py)
  O=gpurun_out/r02u; mkdir -p $O
  timeout 600 python tools/exp_box3.py 10000 > $O/exp_box3.jsonl 2> $O/exp_box3.err
  ;;
v)
  # round 2, call V: specialised single-pivot 3-way epilogue: box rates with / without the epilogue, 3-way GPU tests
  O=gpurun_out/r02v; mkdir -p $O
  timeout 300 python tools/exp_box3.py 10000 "volume 1024" > $O/exp_box3.jsonl 2> $O/exp_box3.err
  timeout 300 python tools/exp_box3.py 10000 "diag pivots [2000" >> $O/exp_box3.jsonl 2>> $O/exp_box3.err
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "3way or czek3 or box or config_shaped or golden" > $O/pytest_3.log 2>&1; echo "rc=$?" >> $O/pytest_3.log
  ;;
w)
  # round 2, call W: w16 thread mapping (no duplicate pivot rewrite) vs the 16 x 16 grid
  O=gpurun_out/r02w; mkdir -p $O
  timeout 300 build/exp_pivot_tma 8192 10000 802819 > $O/exp_pivot_tma_8192.jsonl 2>&1
  timeout 300 build/exp_pivot_tma 4096 20000 802819 > $O/exp_pivot_tma_4096.jsonl 2>&1
  ;;
x)
  # round 2, call X: full GPU suite, cfg2 + cfg4 bench lines, cfg4 launch list (ncu, per-launch times)
  O=gpurun_out/r02x; mkdir -p $O
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
  timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
  timeout 900 python bench.py --steps 5 --warmup 3 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg4.csv python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_cfg4.log 2>&1
  ;;
y)
  # round 2, call Y (4 GPUs): GPU suite incl. NCCL world 2/4, cfg2 / cfg4 at N = 2 / 4 (bench self-launch),
  # cfg4 n_v=3000 launch list on one GPU (share of the two-pivot packed grid)
  O=gpurun_out/r02y; mkdir -p $O
  nvidia-smi topo -m > $O/topo.txt 2>&1
  timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
  timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench_cfg2_n2.json 2> $O/bench_cfg2_n2.err
  timeout 900 python bench.py --gpus 4 --steps 5 --warmup 3 > $O/bench_cfg2_n4.json 2> $O/bench_cfg2_n4.err
  timeout 900 python bench.py --gpus 2 --config cfg4 --steps 2 --warmup 3 > $O/bench_cfg4_n2.json 2> $O/bench_cfg4_n2.err
  timeout 900 python bench.py --gpus 4 --config cfg4 --steps 2 --warmup 3 > $O/bench_cfg4_n4.json 2> $O/bench_cfg4_n4.err
  CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg4_n3000.csv python bench.py --config cfg4 --n-v 3000 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_cfg4_n3000.log 2>&1
  ;;
z)
  # round 2, call Z (2 GPUs): runtime / NCCL tests after the psim_out_t scratch fields, cfg4 N=2 sampled
  # parity from the runtime's scratch box, cfg1 small-problem latency (tools/exp_small.py, bench --config cfg1)
  O=gpurun_out/r02z; mkdir -p $O
  timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_nccl.py -x -q -p no:cacheprovider > $O/pytest_rt.log 2>&1; echo "rc=$?" >> $O/pytest_rt.log
  timeout 900 python bench.py --gpus 2 --config cfg4 --n-v 3000 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/cfg4_n3000_n2.json 2> $O/cfg4_n3000_n2.err
  CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/exp_small.py > $O/exp_small.jsonl 2> $O/exp_small.err
  CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/exp_small.py 1000 2000 >> $O/exp_small.jsonl 2>> $O/exp_small.err
  CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --config cfg1 --steps 20 --warmup 5 > $O/bench_cfg1.json 2> $O/bench_cfg1.err
  ;;
aa)
  # round 2, call AA (4 GPUs): 2-way circulant with the off-diagonal tasks on a second compute stream
  # (no drain between the diagonal grid and the rest): NCCL / runtime tests, cfg2 N=2/4, cfg3 N=4
  O=gpurun_out/r02aa; mkdir -p $O
  timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_nccl.py -x -q -p no:cacheprovider > $O/pytest_rt.log 2>&1; echo "rc=$?" >> $O/pytest_rt.log
  timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu > $O/bench_cfg2_n2.json 2> $O/bench_cfg2_n2.err
  timeout 900 python bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu > $O/bench_cfg2_n4.json 2> $O/bench_cfg2_n4.err
  timeout 1200 python bench.py --gpus 4 --config cfg3 --steps 2 --warmup 3 --no-cpu > $O/bench_cfg3_n4.json 2> $O/bench_cfg3_n4.err
  ;;
bb)
  # round 2, call BB: DRAM bytes per launch of the dominant kernel at the cfg4 and cfg3 bench configs
  # (ncu dram metrics only: one replay pass), for roofline.traffic
  O=gpurun_out/r02bb; mkdir -p $O
  M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
  timeout 1200 ncu --metrics $M --clock-control none -k regex:"k_czek3" -c 16 --csv --log-file $O/traffic_cfg4.csv python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_cfg4.log 2>&1
  timeout 1200 ncu --metrics $M --clock-control none -k regex:"k_minplus2" -c 2 --csv --log-file $O/traffic_cfg3.csv python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_cfg3.log 2>&1
  ;;
cc)
  # round 2, call CC: FP32 2-way tile / inner-op A/B at cfg3's n_f (n_v = 100000), product vs
  # tools/build_variant.sh builds (PSIM_LIB)
  O=gpurun_out/r02cc; mkdir -p $O
  B="python bench.py --config cfg3 --n-v 100000 --steps 2 --warmup 1 --no-cpu --no-e2e --no-parity"
  for r in 1 2; do
    timeout 600 $B > $O/prod_$r.json 2> $O/prod_$r.err
    for v in f32_fadd2 f32_s4 f32_imnmx f32_8x8; do
      PSIM_LIB=build/ab/$v/libpsim.so timeout 600 $B > $O/${v}_$r.json 2> $O/${v}_$r.err
    done
  done
  ;;
z2)
  # round 2, call Z2 (2 GPUs): cfg4 N=2 sampled parity from the runtime's scratch box
  O=gpurun_out/r02z2; mkdir -p $O
  timeout 900 python bench.py --gpus 2 --config cfg4 --n-v 3000 --steps 1 --warmup 1 --no-cpu --no-e2e > $O/cfg4_n3000_n2.json 2> $O/cfg4_n3000_n2.err
  ;;
dd)
  # cfg2 end-to-end breakdown (streamed input, zero-copy values), traced phases
  O=gpurun_out/r02dd; mkdir -p $O
  MODES=1 HV=1 REPS=3 NOCLK=1 timeout 900 python tools/exp_e2e.py > $O/exp_e2e.jsonl 2> $O/exp_e2e.err
  ;;
ee)
  # cfg2 streamed kernel: values to HBM (HV=0) vs zero-copy host (HV=1) vs HBM + per-band D2H
  O=gpurun_out/r02ee; mkdir -p $O
  MODES=1 HV=0 REPS=3 NOCLK=1 timeout 900 python tools/exp_e2e.py > $O/exp_e2e_hv0.jsonl 2> $O/exp_e2e_hv0.err
  PSIM_HOST_OUTPUT=bands MODES=1 HV=1 REPS=3 NOCLK=1 timeout 900 python tools/exp_e2e.py > $O/exp_e2e_bands.jsonl 2> $O/exp_e2e_bands.err
  ;;
ff)
  # the streamed kernel's own duration without upload waits (ncu serialises the copy stream first)
  O=gpurun_out/r02ff; mkdir -p $O
  MODES=1 HV=1 REPS=1 NOCLK=1 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_minplus2" --csv --log-file $O/streamed.csv python tools/exp_e2e.py > $O/exp_e2e.jsonl 2> $O/exp_e2e.err
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_minplus2" -c 1 --csv --log-file $O/resident.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-parity > $O/bench.log 2>&1
  ;;
gg)
  # FP64 2-way warp grid A/B: 4 x 8 (product) vs 2 x 16 (tools/build_variant.sh f64_map1 -DPSIM_F64_MAP=1)
  O=gpurun_out/r02gg; mkdir -p $O
  B="python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e"
  for r in 1 2; do
    timeout 600 $B > $O/map0_$r.json 2> $O/map0_$r.err
    PSIM_LIB=build/ab/f64_map1/libpsim.so timeout 600 $B > $O/map1_$r.json 2> $O/map1_$r.err
  done
  PSIM_LIB=build/ab/f64_map1/libpsim.so timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_map1.log 2>&1; echo "rc=$?" >> $O/pytest_map1.log
  ;;
hh)
  # FP64 2-way tile A/B on cfg2 with TMA staging: 8x8 4-stage (product) vs 8x4 2 CTAs/SM (4 / 3 stages), 8x8 5-stage
  O=gpurun_out/r02hh; mkdir -p $O
  B="python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e"
  for r in 1 2; do
    timeout 600 $B > $O/prod_$r.json 2> $O/prod_$r.err
    for v in f64_8x4_s4 f64_8x4_s3 f64_8x8_s5; do
      PSIM_LIB=build/ab/$v/libpsim.so timeout 600 $B > $O/${v}_$r.json 2> $O/${v}_$r.err
    done
  done
  ;;
final4)
  # round-end check on 4 GPUs: GPU suite (NCCL world 2 / 4), cfg2 at N = 2 / 4 as the driver runs it
  O=gpurun_out/r02final4; mkdir -p $O
  nvidia-smi topo -m > $O/topo.txt 2>&1
  timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
  timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench_cfg2_n2.json 2> $O/bench_cfg2_n2.err
  timeout 900 python bench.py --gpus 4 --steps 5 --warmup 3 > $O/bench_cfg2_n4.json 2> $O/bench_cfg2_n4.err
  timeout 900 python bench.py --gpus 4 --impl reference --steps 2 --warmup 1 > $O/bench_ref_n4.json 2> $O/bench_ref_n4.err
  ;;
ii)
  # FP32 2-way micro-step unroll A/B at cfg3's n_f with TMA staging (product 4 vs 8 / 2)
  O=gpurun_out/r02ii; mkdir -p $O
  B="python bench.py --config cfg3 --n-v 100000 --steps 2 --warmup 1 --no-cpu --no-e2e --no-parity"
  for r in 1 2; do
    timeout 600 $B > $O/prod_$r.json 2> $O/prod_$r.err
    for v in kku8 kku2; do
      PSIM_LIB=build/ab/$v/libpsim.so timeout 600 $B > $O/${v}_$r.json 2> $O/${v}_$r.err
    done
  done
  ;;
jj)
  # streamed kernel: 64 / 1 / 256 upload chunks (tools/exp_stream_order.py)
  O=gpurun_out/r02jj; mkdir -p $O
  timeout 900 python tools/exp_stream_order.py > $O/exp_stream_order.jsonl 2> $O/exp_stream_order.err
  ;;
kk)
  # streamed column-sum CTAs: prefetching double-buffered fold (product build) vs the round-1 fold
  # (build/ab/sums_v1), streamed kernel speed with 1 / 64 upload chunks; streamed GPU tests
  O=gpurun_out/r02kk; mkdir -p $O
  timeout 900 python tools/exp_stream_order.py > $O/new.jsonl 2> $O/new.err
  PSIM_LIB=build/ab/sums_v1/libpsim.so timeout 900 python tools/exp_stream_order.py > $O/old.jsonl 2> $O/old.err
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "stream or e2e or host or pageable" > $O/pytest_stream.log 2>&1; echo "rc=$?" >> $O/pytest_stream.log
  ;;
final1)
  # round-end check on 1 GPU: GPU suite, smoke, default bench (all legs), reference arm, cfg4 line,
  # launch list of the default bench command
  O=gpurun_out/r02final1; mkdir -p $O
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
  timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
  timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
  timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_launches.log 2>&1
  ;;
final2)
  # 2 GPUs after the streamed-upload change: runtime / NCCL tests, cfg2 N=2 with its e2e legs
  O=gpurun_out/r02final2; mkdir -p $O
  timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_nccl.py -x -q -p no:cacheprovider > $O/pytest_rt.log 2>&1; echo "rc=$?" >> $O/pytest_rt.log
  timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 > $O/bench_cfg2_n2.json 2> $O/bench_cfg2_n2.err
  ;;
ll)
  # cfg2 on one GPU under the circulant plans n_pv = 1/2/4/8 (decomposition cost with the TMA kernels)
  O=gpurun_out/r02ll; mkdir -p $O
  timeout 900 python tools/exp_local_grids.py > $O/local_grids.jsonl 2> $O/local_grids.err
  ;;
mm)
  # ncu --set full of the round-end 3-way single-pivot kernel (interleaved pivot loop + single-pivot
  # epilogue) at a cfg4-shaped box, summarised on the box
  O=gpurun_out/r02mm; mkdir -p $O
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_czek3" -s 0 -c 1 -o $O/czek3_final python bench.py --config cfg4 --n-v 1536 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu_3.log 2>&1
  python tools/ncu_summary.py $O/czek3_final.ncu-rep "k_czek3 single-pivot grid, round-end tree, cfg4 n_f=10000, n_v=1536" > $O/ncu_czek3_final.md 2>&1
  ncu -i $O/czek3_final.ncu-rep --page source --csv --print-source sass > $O/czek3_src.csv 2>/dev/null
  python tools/ncu_stalls.py $O/czek3_src.csv > $O/czek3_stalls.txt 2>&1
  rm -f $O/czek3_src.csv
  du -sm $O; if [ $(du -sm $O | cut -f1) -gt 55 ]; then rm -f $O/*.ncu-rep; fi
  ;;
scale4)
  # round-end cfg3 / cfg5 on 4 GPUs
  O=gpurun_out/r02scale4; mkdir -p $O
  timeout 1500 python bench.py --gpus 4 --config cfg3 --steps 2 --warmup 3 --no-cpu > $O/bench_cfg3_n4.json 2> $O/bench_cfg3_n4.err
  timeout 1500 python bench.py --gpus 4 --config cfg5 --steps 2 --warmup 3 --no-cpu > $O/bench_cfg5_n4.json 2> $O/bench_cfg5_n4.err
  # (the first run of this call had no e2e guard: the cfg5 e2e leg pinned 4 x 80 GB and the host killed the ranks)
  ;;
cfg5n4)
  # cfg5 on 4 GPUs with the e2e host-memory guard
  O=gpurun_out/r02cfg5; mkdir -p $O
  free -g > $O/free.txt
  timeout 1500 python bench.py --gpus 4 --config cfg5 --steps 2 --warmup 3 --no-cpu > $O/bench_cfg5_n4.json 2> $O/bench_cfg5_n4.err
  ;;
par4)
  # 4 GPUs: cfg5 / cfg3 with the larger sampled-parity budget
  O=gpurun_out/r02par4; mkdir -p $O
  timeout 1800 python bench.py --gpus 4 --config cfg5 --steps 2 --warmup 3 --no-cpu > $O/bench_cfg5_n4.json 2> $O/bench_cfg5_n4.err
  timeout 1800 python bench.py --gpus 4 --config cfg3 --steps 2 --warmup 3 --no-cpu > $O/bench_cfg3_n4.json 2> $O/bench_cfg3_n4.err
  ;;
f32ncu)
  # ncu --set full (with source) of the FP32 2-way kernel: where the smem bank-conflict counter comes from
  O=gpurun_out/r02f32ncu; mkdir -p $O
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_minplus2" -s 0 -c 1 -o $O/f32 python bench.py --config cfg3 --n-v 16384 --steps 1 --warmup 1 --no-cpu --no-e2e --no-parity > $O/ncu.log 2>&1
  python tools/ncu_summary.py $O/f32.ncu-rep "k_minplus2 FP32 (cfg3 n_f, n_v=16384), round-end tree" > $O/ncu_f32.md 2>&1
  du -sm $O; if [ $(du -sm $O | cut -f1) -gt 55 ]; then rm -f $O/*.ncu-rep; fi
  ;;
final1b)
  # last 1-GPU check after the bench changes: GPU suite, smoke, default bench
  O=gpurun_out/r02final1b; mkdir -p $O
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
  timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
  ;;
cfg4n24)
  # round-end cfg4 at N = 2 / 4 with the 3-way sampled parity from the runtime scratch boxes
  O=gpurun_out/r02cfg4; mkdir -p $O
  timeout 1500 python bench.py --gpus 4 --config cfg4 --steps 2 --warmup 3 --no-cpu > $O/bench_cfg4_n4.json 2> $O/bench_cfg4_n4.err
  timeout 1500 python bench.py --gpus 2 --config cfg4 --steps 2 --warmup 3 --no-cpu > $O/bench_cfg4_n2.json 2> $O/bench_cfg4_n2.err
  ;;
nn)
  # 3-way harness: per-warp rewrite split between the warps of a pair (named barrier) vs ilv
  O=gpurun_out/r02nn; mkdir -p $O
  timeout 300 build/exp_pivot_tma 8192 10000 1064963 > $O/exp_pivot_tma_8192.jsonl 2>&1
  timeout 300 build/exp_pivot_tma 4096 20000 1064963 > $O/exp_pivot_tma_4096.jsonl 2>&1
  ;;
oo)
  # 3-way single-pivot epilogue: one column's loads in flight (product) vs two (build/ab/epi2)
  O=gpurun_out/r02oo; mkdir -p $O
  for r in 1 2; do
    timeout 300 python tools/exp_box3.py 10000 "volume 1024" >> $O/prod.jsonl 2>> $O/prod.err
    PSIM_LIB=build/ab/epi2/libpsim.so timeout 300 python tools/exp_box3.py 10000 "volume 1024" >> $O/epi2.jsonl 2>> $O/epi2.err
  done
  timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "3way or czek3 or box or config_shaped or golden" > $O/pytest_3.log 2>&1; echo "rc=$?" >> $O/pytest_3.log
  ;;
final1c)
  # last check of the round-end tree: GPU suite, smoke, cfg4 and cfg2 bench lines
  O=gpurun_out/r02final1c; mkdir -p $O
  timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
  timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu > $O/bench_cfg4.json 2> $O/bench_cfg4.err
  timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err
  ;;
*)
  echo "usage: $0 <call: a b c d e f g h i j k l m n o p q r s t u v w x y z aa bb cc z2 dd ee ff gg hh final4 ii jj kk final1 final2 ll mm scale4 cfg5n4 par4 f32ncu final1b cfg4n24 nn oo final1c>"; exit 2
  ;;
esac

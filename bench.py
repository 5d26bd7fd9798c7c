"""Benchmark: elementwise comparisons/s of the Czekanowski engine on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2|cfg3|cfg4|cfg5|cfg1]

Metric (BASELINE.json): comparisons/s = n_f * (#unique tuples) / time
(cli.py:144-146, 244). One "step" = one pass of the hot path over the
config's synthetic input: column sums + the fused min-plus / metric /
compaction / checksum kernel(s), all values written to HBM.

* ``value``: device time (CUDA events on the launching stream, max over
  ranks) with inputs already resident in HBM; inputs (>= 0.5 GB) exceed
  the 126 MB L2, so no flush is needed between steps.
* ``e2e``: the same metric through the public API (``run_2way`` with a
  pinned-host ArraySource-style source): H2D of the inputs, the run, and
  D2H of every value + the checksum inside the timed region. 3-way configs:
  ``run_3way`` from the pinned slab with the checksum read back (cfg4's
  288 GB of values exceed host memory).
* ``roofline``: the dominant kernel's achieved cmp/s over its launch time
  vs the min+add issue peak microbenchmarked in the same process
  (psim_peak_minplus).
* ``cpu_baseline`` / ``--impl reference``: the C restatement of the
  reference's blocked kernel (oracle/psim_oracle.c, kind "port") on all
  host threads over a bounded sample of the same workload.

N > 1 runs under torchrun: the config's vector axis is split over N slabs
(circulant 2-way / tetrahedral 3-way plan, NCCL send/recv of blocks; cfg5
splits the field axis), same total work ("strong").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (arity, precision, n_f, n_v, bits, description)
    "cfg1": (2, "double", 1000, 500, 20, "2-way Czekanowski FP64, num_field=1000, num_vector=500"),
    "cfg2": (2, "double", 20000, 40000, 20,
             "2-way Czekanowski FP64, num_field=20000, num_vector=40000"),
    "cfg3": (2, "single", 50000, 200000, 6,
             "2-way Czekanowski FP32, num_field=50000, num_vector=200000"),
    "cfg4": (3, "double", 10000, 6000, 20,
             "3-way Czekanowski FP64, num_field=10000, num_vector=6000"),
    "cfg5": (2, "double", 2000000, 20000, 20,
             "2-way FP64 field-axis split num_field=2000000, num_vector=20000"),
    # SURVEY 8f row f3 (not a BASELINE config): Sorenson on 0/1 data, bit-packed kernel
    "sor2": (2, "double", 20000, 40000, 1,
             "2-way Sorenson (bit-packed AND+POPC) FP64 0/1 data, num_field=20000, "
             "num_vector=40000"),
}
SEED = 2026
METRIC = "elementwise comparisons/sec (2-way & 3-way, FP64/FP32) at 1/2/4/8 B200 vs roofline"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML; the same counters nvidia-smi reads)


class ClockSampler:
    REASONS = {
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sync_boost": 0x10,
        "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int, period: float = 0.2):
        self.index, self.period = index, period
        self.samples: list[tuple[int, int]] = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - depends on the box
            log(f"[bench] NVML unavailable: {e}")

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((mhz, rs))
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.ok:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread:
            self._thread.join()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        mhz = [m for m, _ in self.samples]
        active = 0
        for _, r in self.samples:
            active |= r
        reasons = [k for k, bit in self.REASONS.items() if active & bit]
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(mhz)}


# ---------------------------------------------------------------------------
# distributed plumbing


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def comparisons(arity, n_f, n_v) -> int:
    return n_f * math.comb(n_v, arity)


# ---------------------------------------------------------------------------
# CPU baseline: the C port of the reference's blocked kernel on all host threads


def cpu_baseline(arity, precision, n_f, target_s: float = 12.0) -> dict:
    from oracle import c_oracle
    from oracle import propsim_np as O

    c_oracle.build()
    dt = np.float64 if precision == "double" else np.float32
    nth = c_oracle.threads()
    nf = min(n_f, 250000)
    # calibrate on a small slice, then size a ~target_s sample
    W = O.random_exact(SEED, nf, 4096, 6, dt, v0=0, v1=256)
    t0 = time.perf_counter()
    c_oracle.mgemm(W, W, nth)
    rate0 = nf * 256 * 256 / (time.perf_counter() - t0)
    side = int(math.sqrt(max(rate0 * target_s / nf, 256 * 256)))
    side = max(256, min(side, 16384)) // 128 * 128
    W = O.random_exact(SEED, nf, 1 << 20, 6, dt, v0=0, v1=side)
    t0 = time.perf_counter()
    c_oracle.mgemm(W, W, nth)
    el = time.perf_counter() - t0
    rate = nf * side * side / el
    if arity == 3:  # a 3-way comparison is one min-plus step of the pivot kernel
        pass
    return {
        "value": rate, "unit": "comparisons/s", "cores": nth, "kind": "port",
        "sample": f"oracle/psim_oracle.c blocked min-plus (mingemm.py:94-117 restated), "
                  f"{precision}, n_f={nf} x {side}x{side} outputs, {nth} threads, {el:.1f} s; "
                  f"kernel rate, records/checksum excluded",
    }


# ---------------------------------------------------------------------------
# our arm


def run_ours(args) -> dict | None:
    import torch
    import torch.distributed as dist

    import paper_1705_08210_b200 as P
    from paper_1705_08210_b200 import device as D
    from paper_1705_08210_b200 import engine2, engine3
    from paper_1705_08210_b200 import _native as N

    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", torch.cuda.current_device())
    arity, precision, n_f, n_v, bits, desc = CONFIGS[args.config]
    if args.n_v:
        n_v = args.n_v
    if args.n_f:
        n_f = args.n_f
    code = D.code_of(precision)
    total_cmp = comparisons(arity, n_f, n_v)

    # roofline denominator: min+add issue rate of the mainloop's instruction mix,
    # microbenchmarked in this process (best of its operand variants)
    import ctypes as C

    peak, peak_clk, peak_var = 0.0, 0.0, None
    for var in ((0, 2) if precision == "double" else (0, 1, 2)):
        cps, cpc = C.c_double(), C.c_double()
        N.call("psim_peak_minplus", code, var, 20000 if precision == "double" else 40000,
               C.byref(cps), C.byref(cpc), D.stream_ptr())
        if cps.value > peak:
            peak, peak_clk, peak_var = cps.value, cpc.value, var
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    issue_limit = 32 if precision == "double" else 64  # cmp/clk/SM: 4 resp. 2 instr/cmp
    if args.config == "sor2":  # AND+POPC: one POPC (16/clk/SM) covers 32 fields
        issue_limit = 512
        peak, peak_clk, peak_var = issue_limit * 148 * 1.965e9, 512.0, "popc-nominal"
    log(f"[bench] min+add peak {precision}: {peak:.4e} cmp/s ({peak_clk:.2f} cmp/clk/SM, "
        f"variant {peak_var})")

    # cfg5 is the field-axis split (n_pf = N, NCCL ordered reduce-scatter of
    # partial numerators); every other config splits the vector axis.
    grid = P.DecompGrid(n_pf=world) if args.config == "cfg5" else P.DecompGrid(n_pv=world)
    spec = P.gen_random_exact(SEED, n_f, n_v, bits)
    prob = P.Problem(arity, n_f, n_v, spec, precision,
                     "sorenson" if args.config == "sor2" else "czekanowski")

    if world > 1:
        from paper_1705_08210_b200 import dist as PD

        if arity == 2:
            runner = PD.Runner2(prob, grid)
        else:
            runner = engine3.Runner3Dist(prob, grid, range(grid.n_st), out_budget=40e9)
    else:
        runner = engine2.Resident2(prob, grid) if arity == 2 else engine3.Resident3(prob, grid)
    runner.setup()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        runner.step()
    barrier()
    sampler = ClockSampler(torch.cuda.current_device())
    st = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kernel_ms = []
    with sampler:
        barrier()
        ev0.record(st)
        for _ in range(args.steps):
            kernel_ms.extend(runner.step(timed=True))
        ev1.record(st)
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    launches = runner.launches_per_step * args.steps
    cks = runner.checksum_hex()

    # dominant kernel: algorithmic comparisons per launch over its event time
    kern_cmp = runner.kernel_cmp_per_launch
    kern_ms = (sum(a.elapsed_time(b) for a, b in kernel_ms) / len(kernel_ms)) if kernel_ms else 0.0
    achieved = kern_cmp / (kern_ms * 1e-3) if kern_ms > 0 else None
    traffic = None
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():  # measured once with ncu (bytes per launch), see profiles/
        entry = json.loads(prof.read_text()).get(f"{args.config}:{world}")
        traffic = entry.get("bytes") if isinstance(entry, dict) else entry

    # end-to-end through the public API with host buffers
    e2e = None
    runner.teardown()
    if not args.no_e2e and arity == 2:
        e2e = e2e_2way(P, prob, grid, precision, args, total_cmp, world, rank)
    elif not args.no_e2e and arity == 3:
        e2e = e2e_3way(P, prob, grid, precision, args, total_cmp, world, rank)

    line = None
    if rank == 0:
        clocks = sampler.summary()
        line = {
            "metric": METRIC,
            "value": total_cmp / (ms * 1e-3),
            "unit": "comparisons/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64" if precision == "double" else "f32",
            "data": f"synthetic gen_random_exact(seed={SEED}, bits={bits}) generated in HBM",
            "config": {
                "workload": desc, "arity": arity, "num_field": n_f, "num_vector": n_v,
                "comparisons_per_step": total_cmp,
                "parallelism": ("single slab" if world == 1 else
                                f"field split n_pf={world}" if args.config == "cfg5" else
                                f"circulant n_pv={world}" if arity == 2 else
                                f"tetrahedral n_pv={world}"),
                "l2": "inputs > 126 MB L2 (no flush needed)",
                "checksum": cks,
            },
            "roofline": {
                "bound": "cuda-core",
                "achieved": achieved,
                "peak": peak,
                "unit": "comparisons/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": traffic,
                "kernel": runner.kernel_name,
                "peak_source": ("nominal: POPC issue limit 16/clk/SM x 32 fields at 1965 MHz"
                                if args.config == "sor2" else
                                "measured: psim_peak_minplus microbenchmark of the mainloop "
                                f"instruction mix, same run ({peak_clk:.2f} cmp/clk/SM, "
                                f"variant {peak_var})"),
                "whole_step_frac": (total_cmp / (ms * 1e-3) / world) / peak,
                "issue_limit_cmp_per_clk_sm": issue_limit,
                "frac_of_issue_limit": (achieved / (issue_limit * sm_count * 1e6
                                                    * clocks["sm_mhz"]))
                if achieved and clocks.get("sm_mhz") else None,
            },
            "clocks": clocks,
            "gpu_launches": launches,
        }
        if e2e:
            line["e2e"] = e2e
        if not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline(arity, precision, n_f)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return line


def e2e_2way(P, prob, grid, precision, args, total_cmp, world, rank) -> dict:
    """run_2way through the public API with this rank's input slab in pinned
    host memory: every step copies the slab H2D, runs, and streams every value
    this rank owns back D2H (host_values=True), plus the checksum gather.
    Wall time per step, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1705_08210_b200 import device as D
    from paper_1705_08210_b200.domain import coords_of_rank

    coords = coords_of_rank(rank, grid)
    blk = D.load_block(prob, grid, coords, torch.device("cuda"))  # same synthetic slab
    host = torch.empty((blk.n_vp, blk.n_fp), dtype=blk.data.dtype, pin_memory=True)
    host.copy_(blk.data[:, :blk.n_fp])
    del blk
    src = SlabSource(host.numpy().T, coords)
    e2e_prob = P.Problem(2, prob.n_f, prob.n_v, src, precision)
    transport = "nccl" if world > 1 else "local"
    steps = max(1, min(args.steps, 3))

    def once():
        res = P.run_2way(e2e_prob, grid, transport=transport, host_values=True)
        if world == 1:
            _ = res.records.values  # canonical host array (already copied during the run)
        return res.checksum.hex

    once()  # warm-up (allocations, pinned host buffers)
    times = []
    for _ in range(steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cks = once()
        times.append(time.perf_counter() - t0)
    el = statistics.median(times)
    if world > 1:
        t = torch.tensor([el], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    isz = 8 if precision == "double" else 4
    return {"value": total_cmp / el, "unit": "comparisons/s",
            "h2d_bytes_per_step": prob.n_f * prob.n_v * isz,
            "d2h_bytes_per_step": math.comb(prob.n_v, 2) * isz + 32 * world,
            "seconds_per_step": el, "checksum": cks,
            "values_path": ("zero-copy: the fused kernel stores every value into pinned host "
                            "memory" if os.environ.get("PSIM_HOST_OUTPUT", "direct") != "bands"
                            else "row bands in HBM, D2H copies overlapped with the next band"),
            "api": f"paper_1705_08210_b200.run_2way(Problem(2, n_f, n_v, pinned slab source), "
                   f"grid, transport='{transport}', host_values=True)"}


def e2e_3way(P, prob, grid, precision, args, total_cmp, world, rank) -> dict:
    """run_3way through the public API with this rank's input slab in pinned
    host memory: every step copies the slab H2D (and, under NCCL, circulates
    the blocks), runs every box, and reads back the checksum words. cfg4's
    C(6000, 3) values are 288 GB -- more than host memory -- so they stay
    reduced to the 128-bit checksum on the device (keep_values=False).
    Wall time per step, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1705_08210_b200 import device as D
    from paper_1705_08210_b200.domain import coords_of_rank

    coords = coords_of_rank(rank, grid)
    blk = D.load_block(prob, grid, coords, torch.device("cuda"))
    host = torch.empty((blk.n_vp, blk.n_fp), dtype=blk.data.dtype, pin_memory=True)
    host.copy_(blk.data[:, :blk.n_fp])
    del blk
    src = SlabSource(host.numpy().T, coords)
    e2e_prob = P.Problem(3, prob.n_f, prob.n_v, src, precision)
    transport = "nccl" if world > 1 else "local"
    steps = max(1, min(args.steps, 2))

    def once():
        return P.run_3way(e2e_prob, grid, transport=transport, keep_values=False).checksum.hex

    once()  # warm-up (allocations)
    times = []
    for _ in range(steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cks = once()
        times.append(time.perf_counter() - t0)
    el = statistics.median(times)
    if world > 1:
        t = torch.tensor([el], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    isz = 8 if precision == "double" else 4
    return {"value": total_cmp / el, "unit": "comparisons/s",
            "h2d_bytes_per_step": prob.n_f * prob.n_v * isz,
            "d2h_bytes_per_step": 32 * world,
            "seconds_per_step": el, "checksum": cks,
            "values_path": "reduced on the device to the 128-bit checksum (values exceed host "
                           "memory)",
            "api": f"paper_1705_08210_b200.run_3way(Problem(3, n_f, n_v, pinned slab source), "
                   f"grid, transport='{transport}', keep_values=False)"}


class SlabSource:
    """One rank's input slab in pinned host memory (an ArraySource restricted
    to the caller's own block, reference tests/conftest.py:17-26)."""

    def __init__(self, matrix, coords):
        self.matrix, self.coords = matrix, tuple(coords)

    def local_block(self, problem, grid, coords):
        assert tuple(coords) == self.coords, "slab source holds one rank's block"
        return self.matrix


# ---------------------------------------------------------------------------
# reference arm


def run_reference(args) -> dict | None:
    world, rank, _ = dist_env()
    if rank != 0:
        return None
    arity, precision, n_f, n_v, bits, desc = CONFIGS[args.config]
    total = comparisons(arity, n_f, n_v)
    rates = []
    base = None
    for _ in range(max(1, args.warmup // 3)):
        cpu_baseline(arity, precision, n_f, target_s=3.0)
    for _ in range(max(1, min(args.steps, 3))):
        base = cpu_baseline(arity, precision, n_f, target_s=10.0)
        rates.append(base["value"])
    rate = statistics.median(rates)
    return {
        "impl": "reference",
        "metric": METRIC, "value": rate, "unit": "comparisons/s", "n_gpus": world,
        "steps": len(rates), "warmup": args.warmup, "ms_per_step": total / rate * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if precision == "double" else "f32",
        "data": f"synthetic gen_random_exact(seed={SEED}) sample",
        "config": {"workload": desc, "arity": arity, "num_field": n_f, "num_vector": n_v},
        "cpu_baseline": {**base, "value": rate},
        "e2e": {"value": rate, "unit": "comparisons/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--n-v", type=int, default=0)
    ap.add_argument("--n-f", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    # Keep stdout to the single JSON line: libraries (NCCL's version banner,
    # torch warnings) write to fd 1, so point fd 1 at stderr while running.
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        line = run_reference(args) if args.impl == "reference" else run_ours(args)
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

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


def cpu_baseline(arity, precision, n_f, bits, target_s: float = 12.0) -> dict:
    """The reference's single-rank run_2way (metrics2.py:108-171: dense
    numerator of the diagonal block by the blocked kernel, column sums, the
    value of every pair and the 128-bit checksum) restated in C
    (oracle/psim_oracle.c oracle_czek2_*), on all host threads, over a
    bounded sample of the workload: the config's n_f and dtype, n_v sized
    to take about ``target_s`` seconds. A 3-way comparison is one min-plus
    step as well (metrics3.py:161-169 runs the same blocked kernel), so the
    same sample measures the CPU's comparison rate for both arities.
    The rate is extrapolated to the full config (``extrapolated``)."""
    from oracle import c_oracle
    from oracle import propsim_np as O

    c_oracle.build()
    dt = np.float64 if precision == "double" else np.float32
    nth = c_oracle.threads()
    nf = min(n_f, 250000)
    # calibrate on a small run, then size the sample
    V = O.random_exact(SEED, nf, 1 << 20, bits, dt, v0=0, v1=256)
    t0 = time.perf_counter()
    c_oracle.czek2(V, nth)
    rate0 = nf * 256 * 256 / (time.perf_counter() - t0)
    side = int(math.sqrt(max(rate0 * target_s / nf, 256 * 256)))
    side = max(256, min(side, 16384)) // 128 * 128
    V = O.random_exact(SEED, nf, 1 << 20, bits, dt, v0=0, v1=side)
    t0 = time.perf_counter()
    _, cks, _ = c_oracle.czek2(V, nth)
    el = time.perf_counter() - t0
    # unique pairs are the reference's metric (cli.py:244); the dense
    # diagonal block it computes to get them is its cost
    rate = nf * math.comb(side, 2) / el
    t0 = time.perf_counter()
    c_oracle.mgemm(V, V, nth)
    el_k = time.perf_counter() - t0
    return {
        "value": rate, "unit": "comparisons/s", "cores": nth, "kind": "port",
        "extrapolated": True, "sample_wall_s": el,
        "sample": f"oracle/psim_oracle.c full single-rank run_2way (metrics2.py:108-171 "
                  f"restated: dense blocked min-plus mingemm.py:94-117, column sums, every "
                  f"pair value, 128-bit checksum), {precision}, n_f={nf} x n_v={side} "
                  f"({math.comb(side, 2)} pairs), {nth} threads, {el:.1f} s; rate "
                  f"extrapolated to the full config",
        "kernel_only": {"value": nf * side * side / el_k, "unit": "comparisons/s",
                        "seconds": el_k,
                        "sample": f"blocked min-plus alone, {side}x{side} dense outputs"},
        "sample_checksum": cks,
    }


def cpu_cfg1_end_to_end(expect: str | None) -> dict:
    """cfg1 (2-way FP64, 1000 x 500, seed 2026,
    bits 20) run whole by the C restatement of the reference's single-rank
    run_2way on all host threads; its checksum must equal the reference's
    (SURVEY Appendix B, ea23ebab...) and the GPU's."""
    from oracle import c_oracle
    from oracle import propsim_np as O

    V = O.random_exact(SEED, 1000, 500, 20)
    nth = c_oracle.threads()
    c_oracle.czek2(V, nth)
    times = []
    for _ in range(5):
        t0 = time.perf_counter()
        _, cks, _ = c_oracle.czek2(V, nth)
        times.append(time.perf_counter() - t0)
    el = statistics.median(times)
    return {"workload": CONFIGS["cfg1"][5], "seconds": el,
            "value": 1000 * math.comb(500, 2) / el, "unit": "comparisons/s", "cores": nth,
            "checksum": cks, "checksum_matches_reference": cks == CFG1_REFERENCE_CHECKSUM,
            "checksum_matches_gpu": (cks == expect) if expect else None}


# SURVEY Appendix B / tests/golden/golden.json: the reference's own cfg1 checksum
CFG1_REFERENCE_CHECKSUM = "ea23ebab734aeaaefdc87babae741b72"


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
    # the production mainloop itself over shared-memory operands (variant 3):
    # what the kernel's instruction stream can reach without staging / epilogue
    ml_cps, ml_cpc = C.c_double(), C.c_double()
    N.call("psim_peak_minplus", code, 3, 20000 if precision == "double" else 40000,
           C.byref(ml_cps), C.byref(ml_cpc), D.stream_ptr())
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
        runner = RuntimeBench(prob, grid)
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
        N.launch_count(reset=True)
        ev0.record(st)
        for _ in range(args.steps):
            kernel_ms.extend(runner.step(timed=True))
        ev1.record(st)
        launches = N.launch_count()  # libpsim's own count of the kernels it launched
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms, launches], device=dev, dtype=torch.float64)
        dist.all_reduce(t[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)  # whole job: every rank's launches
        ms, launches = float(t[0].item()), int(t[1].item())
    cks = runner.checksum_hex()
    # checker (after the timed region): sampled tuples recomputed from their
    # columns alone by the oracle (SURVEY 8d "Parity at full size")
    parity = sampled_parity(runner, prob, bits, world, dev) if not args.no_parity else None

    # dominant kernel: algorithmic comparisons per launch over its event time
    if hasattr(runner, "kernel_seconds"):  # the runtime timed its own launches
        kern_cmp = runner.my_cmp * runner.runs / max(1, runner.kernel_grids)
        kern_ms = runner.kernel_seconds * 1e3 / max(1, runner.kernel_grids)
    else:
        kern_cmp = runner.kernel_cmp_per_launch
        kern_ms = (sum(a.elapsed_time(b) for a, b in kernel_ms) / len(kernel_ms)
                   if kernel_ms else 0.0)
    achieved = kern_cmp / (kern_ms * 1e-3) if kern_ms > 0 else None
    traffic = None
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():  # measured once with ncu (bytes per launch), see profiles/
        entry = json.loads(prof.read_text()).get(f"{args.config}:{world}")
        traffic = entry.get("bytes") if isinstance(entry, dict) else entry

    # end-to-end through the public API with host buffers
    e2e = None
    runner.teardown()
    skip = None if args.no_e2e else e2e_host_shortfall(prob, grid, world)
    if skip:
        e2e = {"skipped": skip}
        log(f"[bench] e2e skipped: {skip}")
    elif not args.no_e2e and arity == 2:
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
                "mainloop_ceiling": {
                    "value": ml_cps.value, "cmp_per_clk_sm": ml_cpc.value,
                    "frac": (achieved / ml_cps.value) if achieved and ml_cps.value else None,
                    "what": "psim_peak_minplus variant 3: the production micro_step loop "
                            "over operands resident in shared memory (no staging, no epilogue)"},
                "issue_limit_cmp_per_clk_sm": issue_limit,
                "frac_of_issue_limit": (achieved / (issue_limit * sm_count * 1e6
                                                    * clocks["sm_mhz"]))
                if achieved and clocks.get("sm_mhz") else None,
            },
            "clocks": clocks,
            "gpu_launches": launches,
            "gpu_launches_source": "psim_launch_count (libpsim counts every kernel it "
                                   "launches) over the timed region, summed over ranks",
        }
        if parity is not None:
            line["parity"] = parity
        if e2e:
            line["e2e"] = e2e
        if not args.no_cpu:
            try:
                line["cpu_baseline"] = cpu_baseline(arity, precision, n_f, bits)
            except Exception as e:  # noqa: BLE001 -- reported in the line
                line["cpu_baseline"] = {"error": f"{type(e).__name__}: {e}"}
                log(f"[bench] cpu baseline failed: {e}")
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return line


class RuntimeBench:
    """Multi-GPU harness: each step is ONE psim_run2 / psim_run3 call of the
    run-level runtime (csrc/runtime.cu) on this rank's block resident in HBM:
    validation, column sums, NCCL block exchanges / field reduce-scatter, the
    fused kernels, and the global totals gather. The runtime times its own
    min-plus launches with CUDA events on the launching stream."""

    kernel_name = "k_minplus2 / k_czek3 launch groups inside psim_run2 / psim_run3"

    def __init__(self, prob, grid):
        import torch.distributed as dist

        self.prob, self.grid = prob, grid
        self.world, self.rank = dist.get_world_size(), dist.get_rank()
        self.kernel_seconds, self.kernel_grids, self.runs = 0.0, 0, 0

    def setup(self) -> None:
        import torch

        from paper_1705_08210_b200 import device as D
        from paper_1705_08210_b200 import runtime
        from paper_1705_08210_b200.domain import coords_of_rank

        dev = torch.device("cuda", torch.cuda.current_device())
        c = coords_of_rank(self.rank, self.grid)
        self.block = D.load_block(self.prob, self.grid, c, dev)
        a3 = self.prob.arity == 3
        self.run = runtime.Run(self.prob, self.grid, keep_values=not a3, scratch_values=a3,
                               world=self.world, rank=self.rank, device_block=self.block)
        # comparisons of this rank's min-plus launches: n_fp per element of every
        # whole task / box it computes (a field split computes whole tasks over
        # its field slab and then keeps one chunk of the reduced values)
        from paper_1705_08210_b200.plan import Box, box_count

        self.run.step()
        whole = 0
        for pc in self.run.outcome().pieces:
            if hasattr(pc, "diagonal"):
                whole += pc.m * (pc.m - 1) // 2 if pc.diagonal else pc.m * pc.n
            else:
                whole += box_count(Box((0, 0, 0), pc.i0, pc.i1, pc.j0, pc.j1, pc.k0, pc.k1))
        self.my_cmp = (self.prob.n_f // self.grid.n_pf) * whole

    def step(self, timed: bool = False) -> list:
        out = self.run.step()
        if timed:
            self.kernel_seconds += out.kernel_seconds
            self.kernel_grids += out.kernel_grids
            self.runs += 1
        return []

    @property
    def pieces(self):
        return self.run.outcome().pieces

    def scratch_box(self):
        """3-way: (BoxPiece, device tensor) of the box whose values the
        runtime's scratch buffer still holds after the last step
        (psim_out_t.scratch_piece / scratch_vals), or None."""
        import torch

        from paper_1705_08210_b200.plan import Box, box_count

        out = self.run.out
        if out is None or out.scratch_piece < 0 or not out.scratch_vals:
            return None
        pc = self.run.outcome().pieces[out.scratch_piece]
        n = box_count(Box((0, 0, 0), pc.i0, pc.i1, pc.j0, pc.j1, pc.k0, pc.k1))
        typestr = "<f8" if self.prob.precision == "double" else "<f4"

        class _View:  # the scratch values as a CUDA array (no copy)
            __cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                        "data": (out.scratch_vals, False), "version": 3}

        return pc, torch.as_tensor(_View(), device=torch.device("cuda",
                                                                torch.cuda.current_device()))

    def checksum_hex(self) -> str:
        out = self.run.out
        return format((out.checksum[1] << 64) | out.checksum[0], "032x")

    def teardown(self) -> None:
        import torch

        del self.run, self.block
        torch.cuda.empty_cache()


def sampled_parity(runner, prob, bits, world, dev) -> dict:
    """Checker, run after the timed region (see _local_parity). A checker that
    raises is reported in the line ("checker_errors", "how") instead of
    ending the bench, and every rank still joins the sum over ranks."""
    import torch

    try:
        sampled, mismatches, how = _local_parity(runner, prob, bits)
        errors = 0
    except Exception as e:  # noqa: BLE001 -- reported, not swallowed
        sampled, mismatches, errors = 0, 0, 1
        how = f"checker failed on rank {os.environ.get('RANK', '0')}: {type(e).__name__}: {e}"
        log(f"[bench] parity checker failed: {how}")
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([sampled, mismatches, errors], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        sampled, mismatches, errors = (int(x) for x in t.tolist())
    out = {"sampled": sampled, "mismatches": mismatches, "bitwise": True, "how": how}
    if errors:
        out["checker_errors"] = errors
    return out


def _local_parity(runner, prob, bits) -> tuple:
    """Checker, run after the timed region: tuples of the benchmarked run
    recomputed from their own columns by the oracle (SURVEY 8d "Parity at
    full size": pair_numerators / column_sums / metric2_value, or the 3-way
    triple recompute) and compared bit for bit with the values the kernels
    wrote. 2-way: per value piece of this rank, a grid of sampled rows x
    sampled columns (so ~10^4 pairs need only a few hundred generated
    columns); 3-way: ~10^4 triples (20 pivots x a 25 x 25 grid) of the
    last pivot chunk (at N > 1: the last box in each rank's runtime scratch).
    Returns this rank's (sampled, mismatches, how)."""
    import torch

    from oracle import propsim_np as O
    from paper_1705_08210_b200 import device as D

    dt = np.float64 if prob.precision == "double" else np.float32
    n_f, n_v = prob.n_f, prob.n_v
    rng = np.random.default_rng(7 + int(os.environ.get("RANK", "0")))
    sampled = mismatches = 0
    how = ""
    if prob.arity == 2:
        pieces = getattr(runner, "pieces", None)
        if pieces is None:  # Resident2: one canonical single-slab piece
            from paper_1705_08210_b200.records import PairPiece

            pieces = [PairPiece(0, 0, n_v, n_v, True, 0, n_v, runner.vals)]
        n_pf = getattr(getattr(runner, "grid", None), "n_pf", 1)
        # sampled rows x sampled columns per piece; the recompute costs
        # ~side^2 * n_f adds, so side shrinks with the field depth (cfg2:
        # 160 x 160 -> ~1.3e4 pairs of the diagonal piece; cfg5 at N = 4: ~63 x 63
        # per rank, ~25 s of numpy on each rank)
        side = int(math.sqrt(8e9 / n_f / max(1, len(pieces))))
        side = max(8, min(160, side))
        for pc in pieces:
            if pc.values is None or pc.r1 <= pc.r0:
                continue
            rows = np.unique(np.concatenate([
                rng.integers(pc.r0, pc.r1, size=side - 2), [pc.r0, pc.r1 - 1]]))
            cols = np.unique(np.concatenate([rng.integers(0, pc.n, size=side - 2), [0, pc.n - 1]]))
            VR = O.random_exact_cols(SEED, n_f, n_v, bits, pc.g_row + rows, dt)
            VC = O.random_exact_cols(SEED, n_f, n_v, bits, pc.g_col + cols, dt)
            want = O.pair_values_grid(VR, VC, n_pf)
            li, lj = np.meshgrid(rows, cols, indexing="ij")
            ok = (li < lj) if pc.diagonal else np.ones_like(li, dtype=bool)
            li, lj, want = li[ok], lj[ok], want[ok]
            if pc.diagonal:
                pos = li * (2 * pc.m - li - 1) // 2 + (lj - li - 1)
                base = pc.r0 * (2 * pc.m - pc.r0 - 1) // 2
            else:
                pos, base = li * pc.n + lj, pc.r0 * pc.n
            idx = torch.as_tensor(pos - base, dtype=torch.int64, device=pc.values.device)
            got = D.to_host(pc.values[idx])
            mismatches += int((got.view(np.uint8).reshape(len(got), -1)
                               != want.view(np.uint8).reshape(len(want), -1)).any(axis=1).sum())
            sampled += len(got)
        how = (f"per value piece: sampled rows x sampled columns ({side} each), values "
               f"recomputed from their columns by oracle.propsim_np.pair_values_grid "
               f"(n_pf={n_pf} ordered fold)")
    elif hasattr(runner, "stage_boxes") or (hasattr(runner, "scratch_box")
                                            and runner.scratch_box() is not None):
        # Resident3: the last pivot chunk is in runner.buf; the multi-GPU
        # runtime: the last box of this rank is in its scratch buffer
        from paper_1705_08210_b200.plan import box_count

        if hasattr(runner, "stage_boxes"):
            box, buf = runner.stage_boxes[-1][-1], runner.buf
        else:
            box, buf = runner.scratch_box()
        off, offs = 0, {}
        for j in range(box.j0, box.j1):
            offs[j] = off
            off += max(0, min(box.i1, j) - box.i0) * max(0, box.k1 - max(box.k0, j + 1))
        assert off == box_count(box)
        # 20 pivots of the chunk x (25 sampled rows x 25 sampled columns) each:
        # ~10^4 triples, recomputed as grids (oracle.triple_values_grid)
        js = [j for j in range(box.j0, box.j1)
              if min(box.i1, j) > box.i0 and box.k1 > max(box.k0, j + 1)]
        js = sorted(set(int(x) for x in rng.choice(js, size=min(20, len(js)), replace=False)))
        for j in js:
            klo = max(box.k0, j + 1)
            ih, kh = min(box.i1, j), box.k1
            rows = np.unique(np.concatenate([rng.integers(box.i0, ih, size=23), [box.i0, ih - 1]]))
            cols = np.unique(np.concatenate([rng.integers(klo, kh, size=23), [klo, kh - 1]]))
            VI = O.random_exact_cols(SEED, n_f, n_v, bits, rows, dt)
            VK = O.random_exact_cols(SEED, n_f, n_v, bits, cols, dt)
            xj = O.random_exact_cols(SEED, n_f, n_v, bits, [j], dt)[:, 0]
            want = O.triple_values_grid(VI, xj, VK).ravel()
            ii, kk = np.meshgrid(rows, cols, indexing="ij")
            pos = offs[j] + (ii - box.i0) * (box.k1 - klo) + (kk - klo)
            got = D.to_host(buf[torch.as_tensor(pos.ravel(), device=buf.device)])
            mismatches += int((got.view(np.uint8).reshape(len(got), -1)
                               != want.view(np.uint8).reshape(len(want), -1)).any(axis=1).sum())
            sampled += len(got)
        how = (f"{len(js)} pivots of the last pivot chunk x (sampled rows x sampled columns), "
               "recomputed from their columns by oracle.propsim_np.triple_values_grid")
    else:  # (still joins the sum over ranks: other ranks may hold values)
        how = "values not retained by this harness on this rank"
    return sampled, mismatches, how


def e2e_host_shortfall(prob, grid, world) -> str | None:
    """The e2e legs pin every rank's input slab (and, 2-way, its values) in
    host memory. None when that fits in min(half the host's available
    memory, 256 GB) across the ranks of this node, else the reason to skip
    them: cfg5 at N = 4 would pin 4 x 80 GB, and on the B200 box that got
    its ranks killed by the host (profiles/r02_final/scale4/); cfg3 at N = 4
    pins 120 GB and runs. Decided from node-wide numbers, so all ranks of a
    node skip together."""
    import psutil

    esz = 8 if prob.precision == "double" else 4
    n_fp, n_vp = prob.n_f // grid.n_pf, prob.n_v // grid.n_pv
    tuples = math.comb(prob.n_v, prob.arity)
    per_rank = n_fp * n_vp * esz + (tuples * esz // world if prob.arity == 2 else 0)
    local = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    limit = min(psutil.virtual_memory().available // 2, 256 << 30)
    if per_rank * local > limit:
        return (f"pinned host buffers {per_rank * local / 1e9:.0f} GB on this node > "
                f"{limit / 1e9:.0f} GB (min of half the available memory and 256 GiB)")
    return None


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
    pageable = None
    if world == 1 and not args.no_pageable:
        # the same run from a plain numpy (pageable) block -- the reference's
        # ArraySource (tests/conftest.py:17-26): staged through a pinned ring
        # chunk by chunk under the streamed kernel
        src_p = SlabSource(np.asfortranarray(host.numpy().T.copy()), coords)
        prob_p = P.Problem(2, prob.n_f, prob.n_v, src_p, precision)
        P.run_2way(prob_p, grid, transport=transport, host_values=True)  # warm-up
        tp = []
        for _ in range(steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = P.run_2way(prob_p, grid, transport=transport, host_values=True)
            tp.append(time.perf_counter() - t0)
            assert res.checksum.hex == cks
        pageable = {"value": total_cmp / statistics.median(tp), "unit": "comparisons/s",
                    "seconds_per_step": statistics.median(tp),
                    "api": "run_2way(Problem(2, n_f, n_v, numpy pageable slab source), grid, "
                           "host_values=True)"}
        del src_p, prob_p
    return {"value": total_cmp / el, "unit": "comparisons/s",
            "pageable_source": pageable,
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
    """The reference arm: the reference's own CPU path restated in C
    (oracle/psim_oracle.c; /root/reference is absent on the GPU box) on all
    host threads. Each step is one full single-rank run_2way over a bounded
    sample of the config (same n_f, dtype and bits; values + checksum
    included); the rate is extrapolated to the full config. The line also
    carries cfg1 run whole, checksum-checked."""
    world, rank, _ = dist_env()
    if rank != 0:
        return None
    arity, precision, n_f, n_v, bits, desc = CONFIGS[args.config]
    total = comparisons(arity, n_f, n_v)
    rates, walls = [], []
    base = None
    cpu_baseline(arity, precision, n_f, bits, target_s=2.0)  # warm-up (build, page-in)
    for _ in range(max(1, min(args.steps, 3))):
        base = cpu_baseline(arity, precision, n_f, bits, target_s=10.0)
        rates.append(base["value"])
        walls.append(base["sample_wall_s"])
    rate = statistics.median(rates)
    return {
        "impl": "reference",
        "metric": METRIC, "value": rate, "unit": "comparisons/s", "n_gpus": args.gpus,
        "steps": len(rates), "warmup": 1, "ms_per_step": statistics.median(walls) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if precision == "double" else "f32",
        "data": f"synthetic gen_random_exact(seed={SEED}, bits={bits}) sample",
        "extrapolated": True,
        "extrapolated_full_step_s": total / rate,
        "config": {"workload": desc, "arity": arity, "num_field": n_f, "num_vector": n_v,
                   "sample": base["sample"]},
        "cpu_baseline": {**base, "value": rate},
        "cfg1_end_to_end": cpu_cfg1_end_to_end(None),
        "e2e": {"value": rate, "unit": "comparisons/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def launch_check(args) -> dict | None:
    """--launch-check: the rank plumbing of a bench run without a GPU (gloo):
    every rank reports its rank / world and its slab's plan; rank 0 prints
    them (tests/test_bench_launch.py runs ``bench.py --gpus 2 --launch-check``)."""
    import torch
    import torch.distributed as dist

    from paper_1705_08210_b200 import DecompGrid
    from paper_1705_08210_b200.domain import coords_of_rank
    from paper_1705_08210_b200.plan import Task2, plan_2way

    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    arity, precision, n_f, n_v, bits, desc = CONFIGS[args.config]
    grid = DecompGrid(n_pf=world) if args.config == "cfg5" else DecompGrid(n_pv=world)
    c = coords_of_rank(rank, grid)
    tasks = [e for e in plan_2way(grid, c, n_v // grid.n_pv) if isinstance(e, Task2)]
    mine = torch.tensor([rank, world, len(tasks)], dtype=torch.int64)
    allv = [torch.zeros_like(mine) for _ in range(world)]
    if world > 1:
        dist.all_gather(allv, mine)
        dist.destroy_process_group()
    else:
        allv = [mine]
    if rank != 0:
        return None
    return {"launch_check": True, "n_gpus": world, "gpus_arg": args.gpus,
            "parallelism": (f"field split n_pf={world}" if args.config == "cfg5" else
                            f"circulant n_pv={world}"),
            "ranks": [[int(x) for x in t.tolist()] for t in allv]}


def self_launch(args) -> int | None:
    """``--gpus N`` without a torchrun environment: re-launch this script as
    N ranks (torch.distributed.run, 127.0.0.1) and return their exit code;
    under torchrun, insist that the world size is N. NCCL's init lines
    (communicator, ranks) go to stderr so every run shows its world."""
    world = os.environ.get("WORLD_SIZE")
    if world is not None:
        if int(world) != args.gpus and args.impl == "ours":
            raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
        return None
    if args.gpus <= 1 or args.impl == "reference":
        return None
    import socket
    import subprocess

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    log(f"[bench] self-launch: {' '.join(cmd)}")
    return subprocess.call(cmd, env=env)


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
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-pageable", action="store_true")
    ap.add_argument("--launch-check", action="store_true",
                    help="CPU check of the multi-rank launch (gloo): print the world and plan")
    args = ap.parse_args()
    rc = self_launch(args)
    if rc is not None:
        sys.exit(rc)
    # Keep stdout to the single JSON line: libraries (NCCL's version banner,
    # torch warnings) write to fd 1, so point fd 1 at stderr while running.
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        if args.launch_check:
            line = launch_check(args)
        else:
            line = run_reference(args) if args.impl == "reference" else run_ours(args)
    finally:
        sys.stdout.flush()
        os.dup2(saved, 1)
        os.close(saved)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

"""Small driver for ncu captures and quick kernel timings on the GPU box.

    python tools/prof_driver.py czek2 --precision double --n-v 8192 --n-f 20000 --reps 3
    python tools/prof_driver.py peak  --precision double
    python tools/prof_driver.py czek3 --precision double --n-v 1536 --n-f 10000

Prints one JSON line per repetition with the kernel's CUDA-event time and
comparisons/s (plain run); under ncu the same command is the capture target.
"""
import argparse
import ctypes as C
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1705_08210_b200 as P  # noqa: E402
from paper_1705_08210_b200 import _native as N  # noqa: E402
from paper_1705_08210_b200 import device as D  # noqa: E402
from paper_1705_08210_b200 import engine2, engine3  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kernel", choices=["czek2", "czek3", "peak"])
    ap.add_argument("--precision", default="double")
    ap.add_argument("--n-v", type=int, default=8192)
    ap.add_argument("--n-f", type=int, default=20000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--variant", type=int, default=0)
    a = ap.parse_args()
    code = D.code_of(a.precision)
    if a.kernel == "peak":
        for _ in range(a.reps):
            cps, cpc = C.c_double(), C.c_double()
            N.call("psim_peak_minplus", code, a.variant, 20000, C.byref(cps), C.byref(cpc),
                   D.stream_ptr())
            print(json.dumps({"kernel": "peak", "precision": a.precision, "variant": a.variant,
                              "cmp_per_s": cps.value, "cmp_per_clk_sm": cpc.value}))
        return
    bits = 20 if a.precision == "double" else 6
    prob = P.Problem(2 if a.kernel == "czek2" else 3, a.n_f, a.n_v,
                     P.gen_random_exact(2026, a.n_f, a.n_v, bits), a.precision)
    if a.kernel == "czek2":
        r = engine2.Resident2(prob, P.DecompGrid())
        work = a.n_f * math.comb(a.n_v, 2)
    else:
        r = engine3.Resident3(prob, P.DecompGrid())
        work = a.n_f * math.comb(a.n_v, 3)
    r.setup()
    for _ in range(a.reps):
        ev = r.step(timed=True)
        torch.cuda.synchronize()
        ms = sum(e0.elapsed_time(e1) for e0, e1 in ev)
        print(json.dumps({"kernel": a.kernel, "precision": a.precision, "n_v": a.n_v,
                          "n_f": a.n_f, "ms": ms, "cmp_per_s": work / (ms * 1e-3),
                          "checksum": r.checksum_hex()}))
    r.teardown()


if __name__ == "__main__":
    main()

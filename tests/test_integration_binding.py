"""integration/propsim_b200.py on CPU: B200Result.to_run_result builds the
reference's own RunResult (records in canonical order, Checksum128,
TrafficStats) -- checked against the reference itself when /root/reference
is importable (this container), skipped elsewhere."""
import importlib.util
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = Path("/root/reference/pkg/src")


@pytest.mark.skipif(not REF.exists(), reason="reference not present")
def test_to_run_result_is_the_references(monkeypatch):
    monkeypatch.setenv("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    monkeypatch.syspath_prepend(str(REF))
    from propsim import DecompGrid, Problem, run_2way
    from propsim.verify import checksum, gen_random_exact

    from oracle import propsim_np as O

    spec = importlib.util.spec_from_file_location("propsim_b200",
                                                  ROOT / "integration" / "propsim_b200.py")
    B = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = B  # dataclasses resolve annotations through sys.modules
    spec.loader.exec_module(B)
    n_f, n_v = 40, 12
    prob = Problem(2, n_f, n_v, gen_random_exact(5, n_f, n_v, 6), "double")
    ref = run_2way(prob, DecompGrid())
    vals, cks, deg = O.run_2way(O.random_exact(5, n_f, n_v, 6))[0], None, 0
    # what psim_run2 reports for one rank: one diagonal piece in canonical order
    res = B.B200Result(2, n_v, "double", ref.checksum.value, len(vals), ref.degenerate_count,
                       0.0, np.asarray(vals), [(2, (0, 0, n_v, n_v, 1, 0, n_v, 0), 0, len(vals))],
                       {0: (1, 10, 80)})
    rr = res.to_run_result(prob, DecompGrid())
    assert [r.id.indices for r in rr.records] == [r.id.indices for r in ref.records]
    assert [float(r.value) for r in rr.records] == [float(r.value) for r in ref.records]
    assert checksum(rr.records, n_v) == ref.checksum == rr.checksum
    assert rr.traffic.nbytes == 80 and rr.traffic.by_phase[0] == (1, 10, 80)

"""GPU runs written as metrics directories (row f1): byte-identical to the
directories the reference wrote for the same runs (golden sha256), with the
byte quantisation done on the device (psim_quantize_bytes)."""
import numpy as np
import pytest

from conftest import cuda_available, golden

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device")]


def _run(case, **kw):
    import paper_1705_08210_b200 as P

    if case["kind"] == "uniform":
        src = P.gen_uniform(case["seed"], case["n_f"], case["n_v"])
    else:
        src = P.gen_random_exact(case["seed"], case["n_f"], case["n_v"], case["bits"])
    prob = P.Problem(case["arity"], case["n_f"], case["n_v"], src, case["precision"],
                     case["metric"])
    grid = P.DecompGrid(**case["grid"])
    if case["arity"] == 2:
        return P.run_2way(prob, grid, **kw)
    return P.run_3way(prob, grid, stage=case["stage"], **kw)


@pytest.mark.parametrize("host_values", [False, True])
@pytest.mark.parametrize("case", golden()["outputs"],
                         ids=lambda c: f"{c['arity']}w-{c['precision']}-{c['mode']}-{c['grid']}")
def test_gpu_run_output_matches_reference_directory(case, host_values, tmp_path):
    from paper_1705_08210_b200 import output as OUT
    from test_output import check_directory

    res = _run(case, host_values=host_values)
    OUT.write_run_output(res, OUT.MetricOutputSpec(str(tmp_path), case["mode"]),
                         source={"kind": case["kind"]})
    check_directory(tmp_path, case)


@pytest.mark.parametrize("precision", ["double", "single"])
def test_quantize_kernel_matches_numpy(precision):
    import torch

    from paper_1705_08210_b200 import _native as N
    from paper_1705_08210_b200 import device as D
    from paper_1705_08210_b200.output import quantize_values

    dt = torch.float64 if precision == "double" else torch.float32
    rng = np.random.default_rng(5)
    k = np.arange(256)
    edges = np.concatenate([(k + 0.5) / 255, np.nextafter((k + 0.5) / 255, 0),
                            np.nextafter((k + 0.5) / 255, 1), [-0.0, -3.0, 0.0, 1.0, 2.5]])
    host = np.concatenate([edges, rng.random(100_003) * 1.2 - 0.1]).astype(
        np.float64 if precision == "double" else np.float32)
    dev = torch.from_numpy(host).cuda()
    want = quantize_values(host)
    for off in (0, 1, 3):  # vector and misaligned scalar paths + tails
        v = dev[off:]
        out = torch.empty(v.numel() + 1, dtype=torch.uint8, device="cuda")[1:] if off else \
            torch.empty(v.numel(), dtype=torch.uint8, device="cuda")
        flag = torch.zeros(1, dtype=torch.int64, device="cuda")
        N.call("psim_quantize_bytes", D.code_of(precision), D.ptr(v), v.numel(), D.ptr(out),
               D.ptr(flag), D.stream_ptr())
        assert int(flag.item()) == 0
        assert np.array_equal(out.cpu().numpy(), want[off:])
    bad = dev.clone()
    bad[77] = float("nan")
    out = torch.empty(bad.numel(), dtype=torch.uint8, device="cuda")
    flag = torch.zeros(1, dtype=torch.int64, device="cuda")
    N.call("psim_quantize_bytes", D.code_of(precision), D.ptr(bad), bad.numel(), D.ptr(out),
           D.ptr(flag), D.stream_ptr())
    assert int(flag.item()) == 1


def test_output_needs_values(tmp_path):
    from paper_1705_08210_b200 import output as OUT
    from paper_1705_08210_b200.domain import ConfigError

    case = golden()["outputs"][0]
    res = _run(case, keep_values=False)
    with pytest.raises(ConfigError):
        OUT.write_run_output(res, OUT.MetricOutputSpec(str(tmp_path), "byte"))

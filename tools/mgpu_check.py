"""Multi-GPU parity check (run under torchrun, one process per GPU):

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/mgpu_check.py

Runs run_2way / run_3way with transport="nccl" on several grids whose rank
count equals the world size and compares checksums with the reference's
golden runs (tests/golden/golden.json) and with single-GPU local runs.
Prints one JSON line per case on rank 0; exits non-zero on any mismatch.
"""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1705_08210_b200 as P  # noqa: E402


def check_host_values(world, rank) -> int:
    """run_2way(transport="nccl", host_values=True): every rank's values land in
    pinned host memory (zero-copy from the fused multi-task grids); the values
    each rank holds, with their canonical indices, must re-checksum to the
    global checksum, which must equal the local single-GPU run's."""
    from oracle import propsim_np as O  # test infrastructure: the checker

    n_v = 300 * world + 40
    gen = P.Problem(2, 900, n_v, P.gen_uniform(77, 900, n_v), "double")
    grid = P.DecompGrid(n_pv=world)
    # this rank's slab in pinned host memory: the streamed-input NCCL path
    from paper_1705_08210_b200 import device as D
    from paper_1705_08210_b200.domain import coords_of_rank

    coords = coords_of_rank(rank, grid)
    blk = D.load_block(gen, grid, coords, torch.device("cuda"))
    host = torch.empty((blk.n_vp, blk.n_fp), dtype=blk.data.dtype, pin_memory=True)
    host.copy_(blk.data[:, :blk.n_fp])
    torch.cuda.synchronize()

    class Slab:
        def local_block(self, problem, grid_, coords_):
            assert tuple(coords_) == tuple(coords)
            return host.numpy().T

    prob = P.Problem(2, 900, n_v, Slab(), "double")
    res = P.run_2way(prob, grid, transport="nccl", host_values=True)
    idx = res.records.canonical_indices
    vals = res.records.values
    part = O.checksum(idx, vals) if len(idx) else 0
    t = torch.tensor([part & ((1 << 63) - 1), (part >> 63) & ((1 << 63) - 1), part >> 126],
                     dtype=torch.int64, device="cuda")
    allp = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(allp, t)
    total = sum(int(a[0]) | (int(a[1]) << 63) | (int(a[2]) << 126) for a in allp) % (1 << 128)
    bad = 0
    if rank == 0:
        want = P.run_2way(gen, grid).checksum.hex
        ok = res.checksum.hex == want and format(total, "032x") == want
        bad = int(not ok)
        print(json.dumps({"case": "nccl host_values", "n_v": prob.n_v, "grid": {"n_pv": world},
                          "checksum": res.checksum.hex, "rechecked": format(total, "032x"),
                          "want": want, "ok": ok}), flush=True)
    return bad


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()
    gold = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
    bad = 0
    cases = []
    # golden cases (reference checksums) whose grid fits this world size
    for c in gold["cases"]:
        g = c["grid"]
        if g["n_pf"] * g["n_pv"] * g["n_pr"] != world or "stage" in c or c["kind"] == "matrix":
            continue
        cases.append((c, None))
    # the benchmarked configurations' shapes (reduced n_v) run by the reference
    # (tests/golden/configs.json): cfg2/cfg3 circulant, cfg4 tetrahedral, cfg5
    # field split (its ordered fold on general FP data included)
    conf = json.loads((ROOT / "tests" / "golden" / "configs.json").read_text())
    for c in conf["cases"]:
        g = c["grid"]
        if g["n_pf"] * g["n_pv"] * g["n_pr"] == world:
            cases.append((c, None))
    # extra grids checked against the local single-GPU run
    extra = [
        (2, "double", 1000, 240, dict(n_pv=world)),
        # blocks wider than a column tile: flattened off-diagonal tasks (kCzek2Flat)
        (2, "double", 300, 330 * world, dict(n_pv=world)),
        (2, "single", 200, 200 * world + 8, dict(n_pv=world)),
        (2, "single", 3000, 400, dict(n_pf=world)),
        (2, "double", 777, 120, dict(n_pr=world)),
        (3, "double", 300, 12 * world, dict(n_pv=world)),
        (3, "single", 200, 24, dict(n_pr=world)),
        (3, "double", 200, 24, dict(n_pf=world)),
    ]
    if world % 2 == 0:
        extra.append((2, "double", 500, 96, dict(n_pf=2, n_pv=world // 2)))
        extra.append((3, "double", 64, 24, dict(n_pv=2, n_pr=world // 2)))
        extra.append((3, "single", 300, 24, dict(n_pf=2, n_pv=world // 2)))
    for arity, prec, n_f, n_v, g in extra:
        cases.append((dict(kind="uniform", arity=arity, precision=prec, n_f=n_f, n_v=n_v, seed=31,
                           grid=dict(dict(n_pf=1, n_pv=1, n_pr=1, n_st=1), **g)), "local"))
    for c, mode in cases:
        if c["kind"] == "random-exact":
            src = P.gen_random_exact(c["seed"], c["n_f"], c["n_v"], c["bits"])
        elif c["kind"] == "analytic":
            src = P.gen_analytic(0, c["n_f"], c["n_v"])
        else:
            src = P.gen_uniform(c["seed"], c["n_f"], c["n_v"])
        prob = P.Problem(c["arity"], c["n_f"], c["n_v"], src, c["precision"])
        grid = P.DecompGrid(**c["grid"])
        run = P.run_2way if c["arity"] == 2 else P.run_3way
        res = run(prob, grid, transport="nccl")
        if mode == "local":
            # same grid on one GPU ("local" emulates every rank, incl. the ordered
            # p_f fold, which changes bits vs n_pf=1 on general FP data -- as in
            # the reference)
            want = run(prob, grid).checksum.hex if rank == 0 else None
        else:
            want = c["checksum"]
        if rank == 0:
            ok = res.checksum.hex == want and len(res.records) >= 0
            bad += not ok
            print(json.dumps({"arity": c["arity"], "precision": c["precision"], "n_f": c["n_f"],
                              "n_v": c["n_v"], "grid": c["grid"], "checksum": res.checksum.hex,
                              "want": want, "ok": ok, "elapsed": res.elapsed}), flush=True)
    bad += check_host_values(world, rank)
    bad += check_outputs(gold, world, rank)
    t = torch.tensor([bad], device="cuda")
    dist.broadcast(t, 0)
    dist.destroy_process_group()
    sys.exit(1 if int(t.item()) else 0)


def check_outputs(gold, world, rank) -> int:
    """NCCL runs written as metrics directories (collective write_run_output:
    every process writes its own metrics_<rank>.bin) against the directories
    the reference wrote (golden sha256)."""
    import hashlib
    import tempfile

    from paper_1705_08210_b200 import output as OUT

    bad = 0
    for c in gold["outputs"]:
        g = c["grid"]
        if g["n_pf"] * g["n_pv"] * g["n_pr"] != world:
            continue
        if c["kind"] == "uniform":
            src = P.gen_uniform(c["seed"], c["n_f"], c["n_v"])
        else:
            src = P.gen_random_exact(c["seed"], c["n_f"], c["n_v"], c["bits"])
        prob = P.Problem(c["arity"], c["n_f"], c["n_v"], src, c["precision"], c["metric"])
        grid = P.DecompGrid(**g)
        if c["arity"] == 2:
            res = P.run_2way(prob, grid, transport="nccl")
        else:
            res = P.run_3way(prob, grid, stage=c["stage"], transport="nccl")
        d = [tempfile.mkdtemp(prefix="psim_out_") if rank == 0 else None]
        dist.broadcast_object_list(d, 0)
        OUT.write_run_output(res, OUT.MetricOutputSpec(d[0], c["mode"]),
                             source={"kind": c["kind"]})
        if rank == 0:
            ok = all(hashlib.sha256(Path(d[0], f"metrics_{r}.bin").read_bytes()).hexdigest() == h
                     for r, (_, h) in c["files"].items())
            m = OUT.read_manifest(Path(d[0], "manifest.txt"))
            ok &= all(m[k] == v for k, v in c["manifest"].items()
                      if k not in ("transport", "kernel"))
            bad += not ok
            print(json.dumps({"output": True, "arity": c["arity"], "mode": c["mode"],
                              "grid": g, "stage": c["stage"], "ok": ok}), flush=True)
        dist.barrier()
    return bad


if __name__ == "__main__":
    main()

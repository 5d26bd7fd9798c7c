"""Regenerate the table in profiles/r01_scaling/README.md from its JSON lines.

    python tools/scaling_table.py profiles/r01_scaling
"""
import json
import sys
from pathlib import Path

HEAD = """# Round-1 scaling runs (bench.py, torchrun for N>1; B200)

Each JSON is the single line bench.py printed. cfg2/cfg3/cfg4 keep the same total work at every N
(strong scaling: circulant / tetrahedral vector split); cfg5 is the field split (n_pf = N) and
needs >= 4 GPUs for its 320 GB input. Sweeps marked K/W = 1/1 used 1 warm-up + 1 timed step
(exploratory); 3/3 lines follow the bench contract. `e2e` is the public-API number from pinned
host memory (blank where the sweep ran with --no-e2e).

| workload | N | cmp/s | e2e cmp/s | ms/step | frac (measured peak) | frac (issue limit) | checksum | K/W |
|---|---|---|---|---|---|---|---|---|
"""


def main():
    d = Path(sys.argv[1])
    rows = []
    for f in sorted(d.glob("scale_*.json")):
        j = json.loads(f.read_text().strip().splitlines()[-1])
        e2e = j.get("e2e") if isinstance(j.get("e2e"), dict) else None
        rows.append((j["config"]["workload"], j["n_gpus"], j["value"],
                     e2e["value"] if e2e else None, j["ms_per_step"], j["roofline"]["frac"],
                     j["roofline"].get("frac_of_issue_limit"), j["config"]["checksum"],
                     f"{j['steps']}/{j['warmup']}"))
    rows.sort(key=lambda r: (r[0], r[1]))
    out = [HEAD]
    for w, n, v, e, ms, fr, fi, ck, kw in rows:
        es = f"{e:.4e}" if e else ""
        fis = f"{fi:.3f}" if fi is not None else ""
        out.append(f"| {w} | {n} | {v:.4e} | {es} | {ms:.0f} | {fr:.3f} | {fis} | `{ck}` | {kw} |\n")
    (d / "README.md").write_text("".join(out))


if __name__ == "__main__":
    main()

"""Exact BC (device Brandes) of a config graph vs the estimates of both modes.

    python scripts/exact_bc_check.py c2_rmat18 [out.json]

Prints one JSON line: Brandes kernel time, and max |estimate - exact| for the
deterministic (indexed) and cumulative-epoch (non-det) modes at the config's
(eps, delta).
"""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_1903_09422_b200 import adsamp, datasets
from paper_1903_09422_b200.kadabra import estimate_bc, exact_bc

name = sys.argv[1] if len(sys.argv) > 1 else "c2_rmat18"
w = datasets.CONFIGS[name]
g = datasets.graph(name).graph
t0 = time.perf_counter()
exact, ms = exact_bc(g, device=0)
wall = time.perf_counter() - t0
res = {"config": name, "n": g.num_vertices(), "m": g.num_edges(), "brandes_kernel_s": ms / 1e3, "brandes_wall_s": wall,
       "epsilon": w.epsilon, "delta": w.delta, "max_exact_bc": float(exact.max())}
for label, variant in [("deterministic", adsamp.Variant.indexed), ("nondet_epochs", adsamp.Variant.shared)]:
    cfg = adsamp.EngineConfig(variant=variant, samples_per_frame=1, threads=8, base_seed=42, device=0)
    r = estimate_bc(g, w.epsilon, w.delta, cfg)
    err = np.abs(r.scores - exact)
    res[label] = {"tau": r.tau, "reason": r.reason.name, "max_abs_err": float(err.max()),
                  "argmax_err_vertex": int(err.argmax()), "mean_abs_err": float(err.mean()),
                  "within_eps": bool(err.max() <= w.epsilon)}
line = json.dumps(res)
print(line)
if len(sys.argv) > 2:
    Path(sys.argv[2]).write_text(line + "\n")

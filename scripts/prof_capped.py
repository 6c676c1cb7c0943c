"""Capped estimate_bc on a config (the command ncu wraps for long configs).

    python scripts/prof_capped.py c4_grid 1200 [reps]
"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1903_09422_b200 import adsamp, datasets
from paper_1903_09422_b200.kadabra import estimate_bc

name, cap = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = datasets.CONFIGS[name]
g = datasets.graph(name).graph
cfg = adsamp.EngineConfig(variant=adsamp.Variant[w.variant], samples_per_frame=w.samples_per_frame,
                          base_seed=w.seed, threads=8, device=0, max_cycles=cap)
for i in range(reps):
    t = time.perf_counter()
    r = estimate_bc(g, w.epsilon, w.delta, cfg)
    print(f"{name} cap {cap} rep {i}: tau={r.tau} total={r.run.total_samples} sampler_ms={r.sampler_ms:.2f} "
          f"wall={time.perf_counter()-t:.3f}s E={r.edges_scanned} V={r.vertices_expanded}", flush=True)

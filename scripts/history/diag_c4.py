"""Capped deterministic runs on the C4 grid, reporting sampler errors per path."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1903_09422_b200 import adsamp, datasets
from paper_1903_09422_b200.kadabra import estimate_bc, sample_frames
import numpy as np
g = datasets.graph("c4_grid").graph
print("n", g.num_vertices(), "m", g.num_edges(), flush=True)
for cap in [2000, 20000]:
    cfg = adsamp.EngineConfig(variant=adsamp.Variant.indexed, samples_per_frame=1, base_seed=42, max_cycles=cap, device=0)
    t = time.perf_counter()
    try:
        r = estimate_bc(g, 0.01, 0.1, cfg)
        print(f"cap {cap}: ok tau={r.tau} {time.perf_counter()-t:.2f}s sampler_ms={r.sampler_ms:.1f} E/sample={r.edges_scanned/max(1,r.run.total_samples):.0f} fallbacks={r.store_fallbacks}", flush=True)
    except Exception as e:
        print(f"cap {cap}: {type(e).__name__}: {e} ({time.perf_counter()-t:.2f}s)", flush=True)
# locate failing frames: sample frames in chunks and report which chunk errors
for first in range(0, 20000, 2000):
    try:
        sample_frames(g, 42, 1, first, 2000)
    except Exception as e:
        print(f"frames {first}..{first+2000}: {e}", flush=True)
        for f2 in range(first, first + 2000, 100):
            try:
                sample_frames(g, 42, 1, f2, 100)
            except Exception as e2:
                for f3 in range(f2, f2 + 100):
                    try:
                        sample_frames(g, 42, 1, f3, 1)
                    except Exception:
                        print("  failing frame", f3, flush=True)
                break
        break

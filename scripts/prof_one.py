"""One warm-up + one timed estimate_bc on a config (the command ncu wraps)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1903_09422_b200 import adsamp, datasets
from paper_1903_09422_b200.kadabra import estimate_bc

name = sys.argv[1] if len(sys.argv) > 1 else "c2_rmat18"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = datasets.CONFIGS[name]
g = datasets.graph(name).graph
cfg = adsamp.EngineConfig(variant=adsamp.Variant[w.variant], samples_per_frame=w.samples_per_frame,
                          base_seed=w.seed, threads=8, device=0)
for i in range(reps):
    t = time.perf_counter()
    r = estimate_bc(g, w.epsilon, w.delta, cfg)
    print(f"{name} rep {i}: tau={r.tau} total={r.run.total_samples} ads={r.ads_seconds:.4f}s "
          f"wall={time.perf_counter()-t:.4f}s sampler_ms={r.sampler_ms:.2f} launches={r.kernel_launches} "
          f"E={r.edges_scanned} (rebuild {r.rebuild_edges}, backtrack {r.backtrack_edges}) V={r.vertices_expanded} "
          f"fallbacks={r.store_fallbacks}",
          flush=True)

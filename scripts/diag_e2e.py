"""Break down the e2e step (fresh graph handle per step) on a config."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1903_09422_b200 import adsamp, datasets
from paper_1903_09422_b200.kadabra import estimate_bc
name = sys.argv[1] if len(sys.argv) > 1 else "c2_rmat18"
w = datasets.CONFIGS[name]
g = datasets.graph(name).graph
off, nb = np.ascontiguousarray(g.offsets()), np.ascontiguousarray(g.neighbor_list())
cfg = adsamp.EngineConfig(variant=adsamp.Variant[w.variant], samples_per_frame=1, base_seed=w.seed, threads=8, device=0)
estimate_bc(g, w.epsilon, w.delta, cfg)
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g2 = adsamp.Graph.from_csr(g.num_vertices(), off, nb); t1 = time.perf_counter()
    r = estimate_bc(g2, w.epsilon, w.delta, cfg); t2 = time.perf_counter()
    del g2; torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"from_csr {1e3*(t1-t0):.2f} ms  estimate {1e3*(t2-t1):.2f} ms (pre {1e3*r.preprocess_seconds:.2f} ads {1e3*r.ads_seconds:.2f})  destroy {1e3*(t3-t2):.2f} ms", flush=True)

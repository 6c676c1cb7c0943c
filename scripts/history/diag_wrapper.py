"""Host-side overhead of kadabra.estimate_bc around the device pipeline (ads_seconds)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1903_09422_b200 import adsamp, datasets
from paper_1903_09422_b200.kadabra import estimate_bc
name = sys.argv[1] if len(sys.argv) > 1 else "c3_ba"
w = datasets.CONFIGS[name]
g = datasets.graph(name).graph
cfg = adsamp.EngineConfig(variant=adsamp.Variant[w.variant], samples_per_frame=1, base_seed=w.seed, threads=8, device=0)
for i in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = estimate_bc(g, w.epsilon, w.delta, cfg)
    t1 = time.perf_counter()
    print(f"{name}: wall {1e3*(t1-t0):.2f} ms  ads {1e3*r.ads_seconds:.2f} ms  pre {1e3*r.preprocess_seconds:.3f} ms  sampler {r.sampler_ms:.2f} ms launches {r.kernel_launches}", flush=True)

"""Host timeline of one bench-like C2 step: python call, engine phases (ADSB_TRACE), device events."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1903_09422_b200 import adsamp, datasets
from paper_1903_09422_b200.kadabra import estimate_bc
name = sys.argv[1] if len(sys.argv) > 1 else "c2_rmat18"
w = datasets.CONFIGS[name]
g = datasets.graph(name).graph
cfg = adsamp.EngineConfig(variant=adsamp.Variant[w.variant], samples_per_frame=w.samples_per_frame,
                          base_seed=w.seed, threads=8, device=0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    estimate_bc(g, w.epsilon, w.delta, cfg)
for i in range(4):
    flush.fill_(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    t1 = time.perf_counter()
    r = estimate_bc(g, w.epsilon, w.delta, cfg)
    t2 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    print(f"step {e0.elapsed_time(e1):.3f} ms: record {1e3*(t1-t0):.3f} call {1e3*(t2-t1):.3f} "
          f"(ads {1e3*r.ads_seconds:.3f} pre {1e3*r.preprocess_seconds:.3f} sampler {r.sampler_ms:.3f})", file=sys.stderr, flush=True)

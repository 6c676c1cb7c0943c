"""Where the bench step's time goes beyond the sampler launch (C2, fused epochs)."""
import sys, time
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
for do_flush in (False, True):
    for i in range(4):
        if do_flush:
            flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        e0.record()
        r = estimate_bc(g, w.epsilon, w.delta, cfg)
        e1.record()
        torch.cuda.synchronize()
        print(f"flush={do_flush} step_ms={e0.elapsed_time(e1):.3f} wall_ms={1e3*(time.perf_counter()-t):.3f} "
              f"ads_ms={1e3*r.ads_seconds:.3f} pre_ms={1e3*r.preprocess_seconds:.3f} sampler_ms={r.sampler_ms:.3f}",
              flush=True)

"""Small runs of every sampler path for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1903_09422_b200 import adsamp, datasets
from paper_1903_09422_b200.kadabra import estimate_bc, sample_frames

cases = [("warp", {}, datasets.gen_gnm(600, 2400, 1)),
         ("block", {}, datasets.gen_ba(4000, 4, 3)),
         ("block-global", {"ADSB_NO_SMEM": "1"}, datasets.gen_ba(4000, 4, 3)),
         ("block-lowdeg", {}, datasets.gen_grid(40, 40, 0.1, 3))]
for name, env, pairs in cases:
    os.environ["ADSB_SAMPLER"] = "warp" if name == "warp" else "block"
    for k in ("ADSB_NO_SMEM",):
        os.environ.pop(k, None)
    os.environ.update(env)
    g = adsamp.graph_from_pairs(pairs).graph
    det = estimate_bc(g, 0.1, 0.1, adsamp.EngineConfig(variant=adsamp.Variant.indexed, threads=4, base_seed=3,
                                                          samples_per_frame=1, device=0, max_cycles=300))
    nd = estimate_bc(g, 0.1, 0.1, adsamp.EngineConfig(variant=adsamp.Variant.shared, threads=4, base_seed=3,
                                                         epoch_samples=64, device=0, max_cycles=4))
    fr = sample_frames(g, 5, 1, 0, 50, device=0)
    print(name, det.tau, nd.tau, sum(len(f) for f in fr), flush=True)

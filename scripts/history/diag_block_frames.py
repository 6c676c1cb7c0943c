"""Find frames where the block-team sampler disagrees with the oracle (c1_er)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["ADSB_SAMPLER"] = "block"
import numpy as np
import oracle
from paper_1903_09422_b200 import adsamp, datasets
from paper_1903_09422_b200.kadabra import estimate_bc, sample_frames

pairs = datasets.pairs("c1_er")
pg = adsamp.graph_from_pairs(pairs)
og = oracle.from_pairs(pairs)
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 13
N = 20000
for rep in range(3):
    got = sample_frames(pg.graph, seed, 1, 0, N)
    want = oracle.sample_frames(og, seed, 1, 0, N) if rep == 0 else want
    bad = [i for i in range(N) if not np.array_equal(got[i], want[i])]
    print(f"rep {rep}: {len(bad)} mismatching frames of {N}: {bad[:10]}", flush=True)
    for i in bad[:3]:
        print("  frame", i, "got", got[i].tolist(), "want", want[i].tolist(), flush=True)
for rep in range(10):
    cfg = adsamp.EngineConfig(variant=adsamp.Variant.shared, threads=4, base_seed=13, epoch_samples=64)
    r = estimate_bc(pg.graph, 0.01, 0.1, cfg)
    o = oracle.estimate_bc(og, 0.01, 0.1, mode=oracle.MODE_EPOCH, epoch_samples=64, seed=13) if rep == 0 else o
    d = np.nonzero(r.run.data != o.counts)[0]
    print(f"fused rep {rep}: tau {r.tau}/{o.tau} mismatches {len(d)} at {d[:8].tolist()} "
          f"diff {(r.run.data[d].astype(np.int64) - o.counts[d].astype(np.int64))[:8].tolist()}", flush=True)

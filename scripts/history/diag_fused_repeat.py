"""Repeat the block-team fused-epoch parity check (er100 then c1, B=64) many times."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
os.environ["ADSB_SAMPLER"] = "block"
AUDIT = "/tmp/adsb_audit.bin"
os.environ["ADSB_FUSED_AUDIT"] = AUDIT
import numpy as np
import oracle
from paper_1903_09422_b200 import adsamp, datasets
from paper_1903_09422_b200.kadabra import estimate_bc
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from conftest import SMALL_GRAPHS

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
cases = []
names = [("er100", 0.05), ("c1", 0.01)]
if len(sys.argv) > 3:
    names = [x for x in names if x[0] == sys.argv[3]]
for name, eps in names:
    pairs = datasets.pairs("c1_er") if name == "c1" else SMALL_GRAPHS[name]()
    og = oracle.from_pairs(pairs)
    o = oracle.estimate_bc(og, eps, 0.1, mode=oracle.MODE_EPOCH, epoch_samples=B, seed=13)
    cases.append((name, eps, pairs, o))
frames = {}
bad = 0
for rep in range(reps):
    for name, eps, pairs, o in cases:
        g = adsamp.graph_from_pairs(pairs).graph
        cfg = adsamp.EngineConfig(variant=adsamp.Variant.shared, threads=4, base_seed=13, epoch_samples=B)
        r = estimate_bc(g, eps, 0.1, cfg)
        d = np.nonzero(r.run.data != o.counts)[0]
        if len(d) or r.tau != o.tau:
            bad += 1
            print(f"rep {rep} {name}: tau {r.tau}/{o.tau} mismatches {len(d)} at {d[:8].tolist()} "
                  f"diff {(r.run.data[d].astype(np.int64) - o.counts[d].astype(np.int64))[:8].tolist()} "
                  f"drawn {r.run.total_samples} fallbacks {r.store_fallbacks}", flush=True)
            if name not in frames:
                frames[name] = oracle.sample_frames(oracle.from_pairs(pairs), 13, 1, 0, o.tau)
            miss = set(d.tolist())
            hits = [i for i, fr in enumerate(frames[name]) if len(fr) and set(fr.tolist()) <= miss]
            a = np.fromfile(AUDIT, dtype=np.uint32)
            me = len(a) // (B + 1)
            per, fol = a[: me * B], a[me * B:]
            nep = o.tau // B
            for i in range(nep * B):
                rec, dd = int(per[i] & 0xFFFF), int(per[i] >> 16)
                if rec != len(frames[name][i]):
                    print(f"   sample {i} (epoch {i // B}): recorded {rec} d {dd} expected {len(frames[name][i])} "
                          f"path {frames[name][i].tolist()}", flush=True)
            print(f"   samples whose path lies in the mismatch set: {hits[:10]} (epochs {[h // B for h in hits[:10]]}, "
                  f"last epoch {o.tau // B - 1})", flush=True)
print(f"done: {bad} bad of {len(cases) * reps}")

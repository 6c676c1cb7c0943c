"""Frame parity on dropped-edge grids of growing size, per sampler variant."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import oracle
from paper_1903_09422_b200 import adsamp, datasets
from paper_1903_09422_b200.kadabra import sample_frames

for side in [64, 128, 256, 512]:
    p = datasets.gen_grid(side, side, 0.1, 3)
    og = oracle.from_pairs(p)
    want = oracle.sample_frames(og, 5, 1, 0, 64)
    g = adsamp.graph_from_pairs(p).graph
    try:
        got = sample_frames(g, 5, 1, 0, 64)
        bad = [i for i, (a, b) in enumerate(zip(got, want)) if not np.array_equal(a, b)]
        print(f"grid {side} mode={os.environ.get('ADSB_SAMPLER','auto')} nosmem={os.environ.get('ADSB_NO_SMEM','0')} "
              f"mismatched frames: {bad[:10]} of 64; path lens {[len(x) for x in want[:8]]}", flush=True)
        for i in bad[:2]:
            print("  frame", i, "want", want[i][:12], "... got", got[i][:12], flush=True)
    except Exception as e:
        print(f"grid {side}: ERROR {e}", flush=True)
        break

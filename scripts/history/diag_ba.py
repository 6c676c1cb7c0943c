"""Frame parity on growing BA graphs (set ADSB_NO_SMEM=1 to force the global store)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import oracle
from paper_1903_09422_b200 import adsamp, datasets
from paper_1903_09422_b200.kadabra import sample_frames
sizes = [int(x) for x in sys.argv[1:]] or [1 << 12, 1 << 14, 1 << 16, 1 << 18, 1 << 20]
for n in sizes:
    p = datasets.gen_ba(n, 8, 7)
    og = oracle.from_pairs(p)
    cnt = 200 if n <= (1 << 16) else 40
    want = oracle.sample_frames(og, 42, 1, 0, cnt)
    g = adsamp.graph_from_pairs(p).graph
    try:
        got = sample_frames(g, 42, 1, 0, cnt)
        bad = [i for i, (a, b) in enumerate(zip(got, want)) if not np.array_equal(a, b)]
        print(f"BA n={n} nosmem={os.environ.get('ADSB_NO_SMEM', '0')} mismatches {bad[:8]}", flush=True)
    except Exception as e:
        print(f"BA n={n}: ERROR {e}", flush=True)
        break

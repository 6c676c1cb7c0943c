"""One rank of tests/test_gpu_multirank.py: every case through libadsb's multi-rank
engine over the host transport (gloo). Writes <out_dir>/rank<R>.json."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch.distributed as dist  # noqa: E402

from paper_1903_09422_b200 import adsamp  # noqa: E402
from paper_1903_09422_b200.distributed import Comm  # noqa: E402
from paper_1903_09422_b200.kadabra import estimate_bc  # noqa: E402
from test_gpu_multirank import CASES, config, graph_pairs, summary  # noqa: E402


def main() -> None:
    out_dir = Path(sys.argv[1])
    dist.init_process_group("gloo", init_method="env://")
    rank = dist.get_rank()
    comm = Comm.from_host_group(device=0)
    graphs = {}
    res = {}
    for name, kind, eps, variant, extra in CASES:
        if kind not in graphs:
            graphs[kind] = adsamp.graph_from_pairs(graph_pairs(kind)).graph
        r = estimate_bc(graphs[kind], eps, 0.1, config(variant, extra, comm=comm))
        s = summary(r)
        s.update({"rank": rank, "world": int(r.world)})
        res[name] = s
    (out_dir / f"rank{rank}.json").write_text(json.dumps(res))
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

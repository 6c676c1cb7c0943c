"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Runs oracle/_ref/ref_driver (the unmodified reference headers, compiled by
oracle/Makefile) on seeded graphs written by the product's generators, and
freezes its outputs: run summaries (tau, check_cycles, stop_epoch, omega,
D_ub, reason, FNV-1a of the counts), full count vectors for the small graphs
and C1, and per-frame sampled paths. The graphs themselves are pinned by the
SHA-256 of their edge lists so generator drift is caught.

    python tests/golden/make_golden.py      # needs /root/reference (this container)
"""
from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle  # noqa: E402
from conftest import SMALL_GRAPHS  # noqa: E402
from paper_1903_09422_b200 import datasets  # noqa: E402


def graphs() -> dict[str, np.ndarray]:
    g = {k: np.asarray(v(), dtype=np.uint64).reshape(-1) for k, v in SMALL_GRAPHS.items()}
    g["grid16"] = datasets.gen_grid(16, 16, 0.0, 0)  # the reference's proj/data/grid16.edges layout
    g["grid60_wrap"] = datasets.gen_grid(60, 60, 0.0, 0)  # sigma wraps mod 2^64 on far pairs
    g["ba_small"] = datasets.gen_ba(3000, 3, 5)
    g["rmat12"] = datasets.gen_rmat(12, 8, 0.57, 0.19, 0.19, 3)
    g["c1_er"] = datasets.pairs("c1_er")
    return g


RUNS = [
    # (graph, eps, delta, seed, variant, spf, threads)
    ("c1_er", 0.01, 0.1, 42, "indexed", 1, 8),
    ("c1_er", 0.01, 0.1, 42, "indexed", 1000, 8),
    ("c1_er", 0.02, 0.1, 7, "indexed", 3, 4),
    ("grid16", 0.05, 0.1, 1, "indexed", 1, 4),
    ("grid16", 0.05, 0.1, 1, "indexed", 1000, 4),
    ("er100", 0.05, 0.1, 1000, "indexed", 1, 4),
    ("er100", 0.05, 0.1, 1077, "indexed", 16, 2),
    ("two_components", 0.05, 0.1, 11, "indexed", 5, 1),
    ("star4", 0.05, 0.1, 7, "indexed", 1, 1),
    ("path3", 0.2, 0.1, 7, "indexed", 1, 1),
    ("grid60_wrap", 0.05, 0.1, 3, "indexed", 1, 8),
    ("ba_small", 0.03, 0.1, 9, "indexed", 1, 8),
    ("rmat12", 0.03, 0.1, 9, "indexed", 2, 8),
]

FRAMES = [
    # (graph, seed, spf, first, count)
    ("c1_er", 42, 1, 0, 500),
    ("c1_er", 42, 1000, 3, 2),
    ("grid16", 5, 3, 0, 200),
    ("grid60_wrap", 3, 1, 0, 300),
    ("ba_small", 9, 1, 0, 300),
    ("rmat12", 9, 2, 0, 300),
    ("er24", 31, 1, 0, 200),
]


def main() -> None:
    if not oracle.ref_available():
        oracle.build()
    assert oracle.ref_available(), "needs /root/reference to compile oracle/_ref/ref_driver"
    from paper_1903_09422_b200.datasets import write_edge_list

    gs = graphs()
    out = {"generator": "tests/golden/make_golden.py (oracle/_ref/ref_driver = unmodified reference headers)",
           "graphs": {}, "runs": [], "frames": [], "dub": {}}
    arrays = {}
    with tempfile.TemporaryDirectory() as td:
        paths = {}
        for name, pairs in gs.items():
            path = Path(td) / f"{name}.edges"
            write_edge_list(path, pairs)
            paths[name] = path
            out["graphs"][name] = {"sha256": hashlib.sha256(path.read_bytes()).hexdigest(),
                                   "lines": int(pairs.shape[0] // 2)}
            out["dub"][name] = oracle.ref_dub(path)
        for (gname, eps, delta, seed, variant, spf, threads) in RUNS:
            cpath = Path(td) / "counts.bin"
            r = oracle.ref_run(paths[gname], eps=eps, delta=delta, seed=seed, variant=variant, spf=spf,
                               threads=threads, counts_path=cpath)
            key = f"{gname}|{eps}|{delta}|{seed}|{variant}|{spf}|{threads}"
            counts = np.frombuffer(cpath.read_bytes(), dtype="<u8")
            arrays["counts:" + key] = counts
            r.pop("ads_s"), r.pop("preprocess_s"), r.pop("total_samples"), r.pop("reps", None)
            out["runs"].append({"key": key, "graph": gname, "eps": eps, "delta": delta, "seed": seed,
                                "variant": variant, "spf": spf, "threads": threads, **r})
        for (gname, seed, spf, first, count) in FRAMES:
            fr = oracle.ref_frames(paths[gname], seed=seed, spf=spf, first=first, count=count,
                                   out_path=Path(td) / "frames.bin")
            key = f"{gname}|{seed}|{spf}|{first}|{count}"
            lens = np.array([len(x) for x in fr], dtype=np.uint64)
            arrays["frames_len:" + key] = lens
            arrays["frames_ids:" + key] = np.concatenate(fr).astype(np.uint32) if len(fr) else np.zeros(0, np.uint32)
            out["frames"].append({"key": key, "graph": gname, "seed": seed, "spf": spf, "first": first,
                                  "count": count, "total_ids": int(lens.sum())})
    (HERE / "golden.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    np.savez_compressed(HERE / "golden_arrays.npz", **arrays)
    print(f"wrote {len(out['runs'])} runs, {len(out['frames'])} frame sets")


if __name__ == "__main__":
    main()

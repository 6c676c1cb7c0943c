"""Seeded synthetic stand-ins for BASELINE.json's five configs.

The paper's Appendix-E graphs are not available, so each config is generated
from a fixed seed by libadsb's host generators (csrc/graph_host.cpp) and
restricted to its largest connected component. The edge list is kept in
generation order and ingested with parse_edge_list's first-appearance remap,
so the oracle (reading the written file) and the GPU path see identical ids.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from ._lib import check, lib, u64p
from .adsamp import ParsedGraph, graph_from_pairs


@dataclass(frozen=True)
class Workload:
    name: str
    kind: str
    params: tuple
    epsilon: float
    delta: float
    variant: str
    samples_per_frame: int = 1
    seed: int = 42
    description: str = ""


CONFIGS: dict[str, Workload] = {
    "c1_er": Workload("c1_er", "gnm", (10_000, 50_000, 1), 0.01, 0.1, "indexed", 1, 42,
                      "Erdos-Renyi G(n=10000, m=50000), graph seed 1, LCC; deterministic"),
    "c2_rmat18": Workload("c2_rmat18", "rmat", (18, 16, 0.57, 0.19, 0.19, 11), 0.005, 0.1, "shared", 1, 42,
                          "R-MAT scale 18, ef 16, (.57,.19,.19,.05), graph seed 11, LCC; non-det epochs"),
    "c3_ba": Workload("c3_ba", "ba", (1 << 20, 8, 7), 0.005, 0.1, "indexed", 1, 42,
                      "Barabasi-Albert n=2^20, m=8, seed 7; deterministic"),
    "c4_grid": Workload("c4_grid", "grid", (2048, 2048, 0.1, 3), 0.01, 0.1, "indexed", 1, 42,
                        "2048x2048 lattice, edges dropped w.p. 0.1 (seed 3), LCC; deterministic"),
    "c5_rmat24": Workload("c5_rmat24", "rmat", (24, 16, 0.57, 0.19, 0.19, 24), 0.001, 0.1, "shared", 1, 42,
                          "R-MAT scale 24, ef 16, (.57,.19,.19,.05), graph seed 24, LCC; non-det epochs"),
}


def _take(ptr: u64p, count: int) -> np.ndarray:
    arr = np.ctypeslib.as_array(ptr, shape=(2 * count,)).copy() if count else np.zeros(0, np.uint64)
    lib().adsb_free(ptr)
    return arr


def gen_gnm(n: int, m: int, seed: int, lcc: bool = True) -> np.ndarray:
    p, c = u64p(), C.c_uint64()
    check(lib().adsb_gen_gnm(n, m, seed, int(lcc), C.byref(p), C.byref(c)))
    return _take(p, c.value)


def gen_rmat(scale: int, edge_factor: int, a: float, b: float, c: float, seed: int, lcc: bool = True) -> np.ndarray:
    p, cnt = u64p(), C.c_uint64()
    check(lib().adsb_gen_rmat(scale, edge_factor, a, b, c, seed, int(lcc), C.byref(p), C.byref(cnt)))
    return _take(p, cnt.value)


def gen_ba(n: int, m: int, seed: int) -> np.ndarray:
    p, c = u64p(), C.c_uint64()
    check(lib().adsb_gen_ba(n, m, seed, C.byref(p), C.byref(c)))
    return _take(p, c.value)


def gen_grid(width: int, height: int, p_drop: float, seed: int, lcc: bool = True) -> np.ndarray:
    p, c = u64p(), C.c_uint64()
    check(lib().adsb_gen_grid(width, height, p_drop, seed, int(lcc), C.byref(p), C.byref(c)))
    return _take(p, c.value)


def pairs(name: str) -> np.ndarray:
    w = CONFIGS[name]
    if w.kind == "gnm":
        return gen_gnm(*w.params)
    if w.kind == "rmat":
        return gen_rmat(*w.params)
    if w.kind == "ba":
        return gen_ba(*w.params)
    if w.kind == "grid":
        return gen_grid(*w.params)
    raise KeyError(name)


def write_edge_list(path: str | os.PathLike, p: np.ndarray) -> None:
    a = np.ascontiguousarray(p, dtype=np.uint64)
    check(lib().adsb_write_edge_list(os.fsencode(path), a.ctypes.data_as(u64p), a.shape[0] // 2))


def graph(name: str, cache_dir: str | os.PathLike | None = None) -> ParsedGraph:
    """The config's graph. With a cache directory (argument or ADSB_GRAPH_CACHE)
    the ingested CSR is kept as a binary cache (adsamp.save_graph) and later
    calls load it instead of regenerating (C5: ~30 s -> ~1 s)."""
    from .adsamp import load_graph, save_graph
    d = cache_dir or os.environ.get("ADSB_GRAPH_CACHE")
    if not d:
        return graph_from_pairs(pairs(name))
    path = Path(d) / f"{name}.adsbcsr"
    if path.exists():
        return load_graph(path)
    parsed = graph_from_pairs(pairs(name))
    path.parent.mkdir(parents=True, exist_ok=True)
    save_graph(parsed, path)
    return parsed


def edge_list_file(name: str, directory: str | os.PathLike) -> Path:
    """Write (once) the config's edge list as text for the CPU oracles."""
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    path = d / f"{name}.edges"
    if not path.exists():
        tmp = path.with_suffix(".tmp")
        write_edge_list(tmp, pairs(name))
        tmp.rename(path)
    return path

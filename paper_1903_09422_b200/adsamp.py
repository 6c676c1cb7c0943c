"""Python mirror of the reference's `adsamp` C++ API, backed by libadsb.so.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/adsamp/ (graph.hpp, engine.hpp, rng.hpp); the
KADABRA layer lives in `paper_1903_09422_b200.kadabra` (kadabra.hpp). All
traversal work runs on the GPU through the C ABI; the pure-Python pieces are
the integer RNG helpers and config validation, exactly as small as the
reference's own inline functions.
"""
from __future__ import annotations

import ctypes as C
import enum
import io
import math
import os
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from ._lib import Config, InvalidArgument, ParseError, check, lib, u32p, u64p

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


# --------------------------------------------------------------------------- rng.hpp
def mix64(z: int) -> int:
    """rng.hpp:12-19"""
    z &= MASK64
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & MASK64
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & MASK64
    z ^= z >> 31
    return z


class SplitMix64:
    """rng.hpp:23-48"""

    def __init__(self, seed: int = 0):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + GOLDEN) & MASK64
        return mix64(self.state)

    def next_below(self, bound: int) -> int:
        m = self.next() * bound
        lo = m & MASK64
        if lo < bound:
            threshold = ((1 << 64) - bound) % bound if bound else 0
            while lo < threshold:
                m = self.next() * bound
                lo = m & MASK64
        return m >> 64


def reseed(base_seed: int, frame_index: int) -> int:
    """rng.hpp:53-55"""
    return mix64(base_seed ^ ((frame_index * GOLDEN) & MASK64))


def stream_rng(base_seed: int, frame_index: int) -> SplitMix64:
    """rng.hpp:57-59"""
    return SplitMix64(reseed(base_seed, frame_index))


# --------------------------------------------------------------------------- engine.hpp
class Variant(enum.IntEnum):
    """engine.hpp:63"""
    sequential = 0
    barrier = 1
    local = 2
    shared = 3
    indexed = 4


def to_string(v: Variant) -> str:
    return Variant(v).name


def parse_variant(s: str) -> Variant:
    """engine.hpp:76-83"""
    try:
        return Variant[s]
    except KeyError:
        raise InvalidArgument(f"unknown variant '{s}'") from None


@dataclass
class EngineConfig:
    """engine.hpp:85-106, plus the GPU pipeline knobs (include/adsb.h)."""
    threads: int = 1
    variant: Variant = Variant.local
    frame_groups: int = 2
    check_interval: int = 1000
    latency_exponent: float = 1.33
    samples_per_frame: int = 1000
    bounded_memory: bool = False
    reservation_block: int = 4
    queue_high_water: int = 64
    base_seed: int = 1
    # GPU pipeline
    epoch_samples: int = 0
    max_cycles: int = 0
    device: int = -1
    comm: object | None = None

    def validate(self) -> None:
        if self.threads < 1:
            raise InvalidArgument("threads must be >= 1")
        if self.variant == Variant.shared and not (1 <= self.frame_groups <= self.threads):
            raise InvalidArgument("frame groups must satisfy 1 <= F <= T")
        if self.check_interval < 1:
            raise InvalidArgument("check interval must be >= 1")
        if not self.latency_exponent > 0:
            raise InvalidArgument("xi must be > 0")
        if self.samples_per_frame < 1:
            raise InvalidArgument("samples per frame must be >= 1")
        if self.reservation_block < 1:
            raise InvalidArgument("reservation block must be >= 1")

    def to_c(self) -> Config:
        c = Config()
        lib().adsb_config_init(C.byref(c))
        c.variant = int(self.variant)
        c.threads = self.threads
        c.frame_groups = self.frame_groups
        c.check_interval = self.check_interval
        c.latency_exponent = self.latency_exponent
        c.samples_per_frame = self.samples_per_frame
        c.epoch_samples = self.epoch_samples
        c.base_seed = self.base_seed & MASK64
        c.max_cycles = self.max_cycles
        c.device = self.device
        c.comm = getattr(self.comm, "handle", None)
        c.bounded_memory = int(bool(self.bounded_memory))
        c.reservation_block = self.reservation_block
        c.queue_high_water = self.queue_high_water
        return c


def check_budget(check_interval: int, threads: int, xi: float) -> int:
    """engine.hpp:110-116"""
    out = C.c_uint64()
    check(lib().adsb_check_budget(check_interval, threads, xi, C.byref(out)))
    return out.value


def shared_frame_target(t: int, F: int) -> int:
    """engine.hpp:119"""
    return t % F


def indexed_frame_index(epoch: int, t: int, T: int) -> int:
    """engine.hpp:124-126"""
    return epoch * T + t


class ReservationCounter:
    """engine.hpp:129-131 (single-process claim counter)."""

    def __init__(self):
        self.next_claim = 0


def reserve_indices(counter: ReservationCounter, T: int, a: int) -> list[int]:
    """engine.hpp:137-144"""
    k = counter.next_claim
    counter.next_claim += 1
    out = (C.c_uint64 * (a + 1))()
    check(lib().adsb_reserve_indices(k, T, a, out))
    return list(out)


@dataclass
class QueueStats:
    """engine.hpp:156-161, per sampler team: frames sampled ahead of the in-order
    consumption point (deterministic batches, epoch ring)."""
    max_depth: int = 0
    mean_depth: float = 0.0
    allocated: int = 0
    high_water_exceeded: bool = False


@dataclass
class RunResult:
    """engine.hpp:163-171"""
    data: np.ndarray
    num: int = 0
    total_samples: int = 0
    per_thread_samples: list = field(default_factory=list)
    check_cycles: int = 0
    stop_epoch: int = 0
    queue: QueueStats = field(default_factory=QueueStats)


# --------------------------------------------------------------------------- graph.hpp
def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


class Graph:
    """graph.hpp:29-76: immutable undirected CSR, ascending adjacency.

    Owns an adsb_graph handle; the device replica is created on first use.
    """

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        n = C.c_uint32()
        nnz = C.c_uint64()
        self._destroy = lib().adsb_graph_destroy
        check(lib().adsb_graph_info(self._h, C.byref(n), C.byref(nnz)))
        self._n = n.value
        self._nnz = nnz.value
        self._csr: tuple[np.ndarray, np.ndarray] | None = None

    def __del__(self):
        h = getattr(self, "_h", None)
        destroy = getattr(self, "_destroy", None)
        if h and destroy is not None:  # bound at construction: module globals may be gone at exit
            destroy(h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @staticmethod
    def from_edges(num_vertices: int, edges: Sequence[tuple[int, int]] | np.ndarray) -> "Graph":
        """graph.hpp:35-58"""
        e = _u32(np.asarray(edges, dtype=np.int64).reshape(-1, 2)) if len(edges) else np.zeros((0, 2), np.uint32)
        h = C.c_void_p()
        check(lib().adsb_graph_from_edges(num_vertices, e.ctypes.data_as(u32p), e.shape[0], C.byref(h)))
        return Graph(h)

    @staticmethod
    def from_csr(num_vertices: int, offsets, neighbors) -> "Graph":
        off = _u64(offsets)
        nb = _u32(neighbors)
        if off.shape[0] != num_vertices + 1:
            raise InvalidArgument("offsets must have n+1 entries")
        h = C.c_void_p()
        check(lib().adsb_graph_from_csr(num_vertices, off.ctypes.data_as(u64p), nb.ctypes.data_as(u32p), C.byref(h)))
        return Graph(h)

    def num_vertices(self) -> int:
        return self._n

    def num_edges(self) -> int:
        return self._nnz // 2

    def _load_csr(self) -> tuple[np.ndarray, np.ndarray]:
        if self._csr is None:
            off = np.empty(self._n + 1, dtype=np.uint64)
            nb = np.empty(max(self._nnz, 1), dtype=np.uint32)
            check(lib().adsb_graph_copy_csr(self._h, off.ctypes.data_as(u64p), nb.ctypes.data_as(u32p)))
            self._csr = (off, nb[: self._nnz])
        return self._csr

    def offsets(self) -> np.ndarray:
        return self._load_csr()[0]

    def neighbor_list(self) -> np.ndarray:
        return self._load_csr()[1]

    def neighbors(self, u: int) -> np.ndarray:
        off, nb = self._load_csr()
        return nb[int(off[u]):int(off[u + 1])]

    def degree(self, u: int) -> int:
        off = self.offsets()
        return int(off[u + 1] - off[u])


@dataclass
class ParsedGraph:
    """graph.hpp:80-83"""
    graph: Graph
    original_ids: np.ndarray


def _parsed(h: C.c_void_p) -> ParsedGraph:
    g = Graph(h)
    ids = np.empty(max(g.num_vertices(), 1), dtype=np.uint64)
    check(lib().adsb_graph_copy_original_ids(h, ids.ctypes.data_as(u64p)))
    return ParsedGraph(g, ids[: g.num_vertices()])


def parse_edge_list(src) -> ParsedGraph:
    """graph.hpp:93-131 / :133-136. Accepts a str, bytes or a text stream."""
    if isinstance(src, io.IOBase) or hasattr(src, "read"):
        src = src.read()
    data = src.encode() if isinstance(src, str) else bytes(src)
    h = C.c_void_p()
    check(lib().adsb_graph_parse_text(data, len(data), C.byref(h)))
    return _parsed(h)


def parse_edge_list_file(path: str | os.PathLike) -> ParsedGraph:
    h = C.c_void_p()
    check(lib().adsb_graph_parse_file(os.fsencode(path), C.byref(h)))
    return _parsed(h)


def save_graph(g: "Graph | ParsedGraph", path: str | os.PathLike) -> None:
    """Binary CSR cache of an ingested graph (dense ids, adjacency, original ids)."""
    gg = g.graph if isinstance(g, ParsedGraph) else g
    check(lib().adsb_graph_save(gg.handle, os.fsencode(path)))


def load_graph(path: str | os.PathLike) -> ParsedGraph:
    """Inverse of save_graph: the identical graph, read with parallel I/O and
    checked against its checksum (ParseError when damaged or truncated)."""
    h = C.c_void_p()
    check(lib().adsb_graph_load(os.fsencode(path), C.byref(h)))
    return _parsed(h)


def graph_from_pairs(pairs) -> ParsedGraph:
    """parse_edge_list semantics on (id, id) records already in memory."""
    p = _u64(np.asarray(pairs).reshape(-1))
    if p.shape[0] % 2:
        raise InvalidArgument("pairs must hold an even number of ids")
    h = C.c_void_p()
    check(lib().adsb_graph_from_pairs(p.ctypes.data_as(u64p), p.shape[0] // 2, C.byref(h)))
    return _parsed(h)


def serialize_edge_list(g: Graph) -> str:
    """graph.hpp:140-144"""
    n = C.c_uint64(0)
    check(lib().adsb_graph_serialize(g.handle, None, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib().adsb_graph_serialize(g.handle, buf, C.byref(n)))
    return buf.raw[: n.value].decode()


@dataclass
class ComponentLabels:
    """graph.hpp:146-151"""
    label: np.ndarray
    num_components: int

    def same_component(self, u: int, v: int) -> bool:
        return bool(self.label[u] == self.label[v])


def connected_components(g: Graph, device: int = -1) -> ComponentLabels:
    """graph.hpp:153-175 (computed on the GPU, identical numbering)."""
    lab = np.empty(max(g.num_vertices(), 1), dtype=np.uint32)
    c = C.c_uint32()
    check(lib().adsb_connected_components(g.handle, device, lab.ctypes.data_as(u32p), C.byref(c)))
    return ComponentLabels(lab[: g.num_vertices()], c.value)


def eccentricity(g: Graph, source: int, device: int = -1) -> int:
    """graph.hpp:178-197"""
    out = C.c_uint64()
    check(lib().adsb_eccentricity(g.handle, device, source, C.byref(out)))
    return out.value


def diameter_upper_bound(g: Graph, device: int = -1) -> int:
    """graph.hpp:202-214"""
    out = C.c_uint64()
    check(lib().adsb_diameter_upper_bound(g.handle, device, C.byref(out)))
    return out.value


from . import kadabra  # noqa: E402  (adsamp::kadabra namespace)

__all__ = [
    "mix64", "SplitMix64", "reseed", "stream_rng", "Variant", "to_string", "parse_variant", "EngineConfig",
    "check_budget", "shared_frame_target", "indexed_frame_index", "ReservationCounter", "reserve_indices",
    "RunResult", "Graph", "ParsedGraph", "parse_edge_list", "parse_edge_list_file", "graph_from_pairs",
    "serialize_edge_list", "ComponentLabels", "connected_components", "eccentricity", "diameter_upper_bound",
    "ParseError", "kadabra",
]

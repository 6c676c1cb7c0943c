"""ctypes wrapper of the CPU oracle (oracle.c) and runner of the compiled
reference driver (_ref/ref_driver).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"
REF_DRIVER = HERE / "_ref" / "ref_driver"

MODE_INDEXED, MODE_EPOCH = 0, 1
REASONS = {0: "eps_converged", 1: "omega_reached", 2: "capped"}


class _Graph(C.Structure):
    _fields_ = [("n", C.c_uint32), ("nnz", C.c_uint64), ("offsets", C.POINTER(C.c_uint64)),
                ("nbrs", C.POINTER(C.c_uint32)), ("original_ids", C.POINTER(C.c_uint64))]


class _Config(C.Structure):
    _fields_ = [("mode", C.c_int32), ("nominal_threads", C.c_uint32), ("samples_per_frame", C.c_uint64),
                ("epoch_samples", C.c_uint64), ("seed", C.c_uint64), ("max_frames", C.c_uint64), ("c", C.c_double)]


class _Result(C.Structure):
    _fields_ = [("tau", C.c_uint64), ("check_cycles", C.c_uint64), ("stop_epoch", C.c_uint64),
                ("omega", C.c_uint64), ("diameter_bound", C.c_uint64), ("total_samples", C.c_uint64),
                ("edges_scanned", C.c_uint64), ("vertices_expanded", C.c_uint64), ("reason", C.c_int32),
                ("pad", C.c_int32), ("degenerate_steps", C.c_uint64)]


_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        u64p, u32p = C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)
        gp = C.POINTER(_Graph)
        L.or_next_below.argtypes = [u64p, C.c_uint64]
        L.or_next_below.restype = C.c_uint64
        L.or_reseed.argtypes = [C.c_uint64, C.c_uint64]
        L.or_reseed.restype = C.c_uint64
        L.or_parse_edge_list_text.argtypes = [C.c_char_p, C.c_size_t, gp, C.c_char_p, C.c_size_t]
        L.or_parse_edge_list_file.argtypes = [C.c_char_p, gp, C.c_char_p, C.c_size_t]
        L.or_graph_from_pairs.argtypes = [u64p, C.c_uint64, gp, C.c_char_p, C.c_size_t]
        L.or_graph_from_edges.argtypes = [C.c_uint32, u32p, C.c_uint64, gp, C.c_char_p, C.c_size_t]
        L.or_graph_free.argtypes = [gp]
        L.or_graph_free.restype = None
        L.or_connected_components.argtypes = [gp, u32p]
        L.or_connected_components.restype = C.c_uint32
        L.or_eccentricity.argtypes = [gp, C.c_uint32]
        L.or_eccentricity.restype = C.c_uint64
        L.or_diameter_upper_bound.argtypes = [gp]
        L.or_diameter_upper_bound.restype = C.c_uint64
        L.or_compute_omega.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_double, u64p]
        L.or_f_bound.argtypes = [C.c_double, C.c_double, C.c_uint64, C.c_uint64, C.POINTER(C.c_double)]
        L.or_g_bound.argtypes = [C.c_double, C.c_double, C.c_uint64, C.c_uint64, C.POINTER(C.c_double)]
        L.or_kadabra_check.argtypes = [u64p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_double,
                                       C.POINTER(C.c_int)]
        L.or_scratch_new.argtypes = [C.c_uint32]
        L.or_scratch_new.restype = C.c_void_p
        L.or_scratch_free.argtypes = [C.c_void_p]
        L.or_scratch_free.restype = None
        L.or_sample_frame.argtypes = [gp, u32p, C.c_uint64, C.c_uint64, C.c_uint64, u32p, C.c_uint64, C.c_void_p]
        L.or_sample_frame.restype = C.c_uint64
        L.or_estimate_bc.argtypes = [gp, C.c_double, C.c_double, C.POINTER(_Config), u64p,
                                     C.POINTER(C.c_double), C.POINTER(_Result), C.c_char_p, C.c_size_t]
        L.or_estimate_bc_threads.argtypes = [gp, C.c_double, C.c_double, C.POINTER(_Config), C.c_int, u64p,
                                             C.POINTER(C.c_double), C.POINTER(_Result), C.c_char_p, C.c_size_t]
        L.or_brandes.argtypes = [gp, C.POINTER(C.c_double), C.c_int]
        L.or_brandes.restype = None
        _lib = L
    return _lib


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class Graph:
    """CSR built by the restated parser / from_edges."""

    def __init__(self):
        self._g = _Graph()

    def __del__(self):
        if getattr(self, "_g", None) is not None and self._g.offsets:
            lib().or_graph_free(C.byref(self._g))

    @property
    def n(self) -> int:
        return self._g.n

    @property
    def offsets(self) -> np.ndarray:
        return np.ctypeslib.as_array(self._g.offsets, shape=(self.n + 1,)).copy()

    @property
    def nbrs(self) -> np.ndarray:
        if self._g.nnz == 0:
            return np.zeros(0, np.uint32)
        return np.ctypeslib.as_array(self._g.nbrs, shape=(self._g.nnz,)).copy()

    @property
    def original_ids(self) -> np.ndarray | None:
        if not self._g.original_ids:
            return None
        return np.ctypeslib.as_array(self._g.original_ids, shape=(self.n,)).copy()


def _call(fn, *args) -> Graph:
    g = Graph()
    err = C.create_string_buffer(256)
    rc = fn(*args, C.byref(g._g), err, 256)
    if rc:
        raise OracleError(rc, err.value.decode())
    return g


def parse_text(text: str | bytes) -> Graph:
    data = text.encode() if isinstance(text, str) else text
    return _call(lib().or_parse_edge_list_text, data, len(data))


def parse_file(path) -> Graph:
    return _call(lib().or_parse_edge_list_file, os.fsencode(path))


def from_pairs(pairs) -> Graph:
    p = np.ascontiguousarray(np.asarray(pairs, dtype=np.uint64).reshape(-1))
    return _call(lib().or_graph_from_pairs, p.ctypes.data_as(C.POINTER(C.c_uint64)), p.shape[0] // 2)


def from_edges(n: int, edges) -> Graph:
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1))
    return _call(lib().or_graph_from_edges, n, e.ctypes.data_as(C.POINTER(C.c_uint32)), e.shape[0] // 2)


def components(g: Graph) -> tuple[np.ndarray, int]:
    lab = np.empty(max(g.n, 1), np.uint32)
    c = lib().or_connected_components(C.byref(g._g), lab.ctypes.data_as(C.POINTER(C.c_uint32)))
    return lab[: g.n], c


def eccentricity(g: Graph, s: int) -> int:
    return lib().or_eccentricity(C.byref(g._g), s)


def diameter_upper_bound(g: Graph) -> int:
    return lib().or_diameter_upper_bound(C.byref(g._g))


def compute_omega(dub: int, eps: float, delta: float, c: float = 0.5) -> int:
    out = C.c_uint64()
    rc = lib().or_compute_omega(dub, eps, delta, c, C.byref(out))
    if rc:
        raise OracleError(rc, "epsilon and delta must lie in (0,1)")
    return out.value


def f_bound(b, delta_v, omega, tau) -> float:
    out = C.c_double()
    rc = lib().or_f_bound(b, delta_v, omega, tau, C.byref(out))
    if rc:
        raise OracleError(rc, "domain")
    return out.value


def g_bound(b, delta_v, omega, tau) -> float:
    out = C.c_double()
    rc = lib().or_g_bound(b, delta_v, omega, tau, C.byref(out))
    if rc:
        raise OracleError(rc, "domain")
    return out.value


def kadabra_check(data, num: int, omega: int, eps: float, delta_v: float) -> bool:
    d = np.ascontiguousarray(np.asarray(data, dtype=np.uint64))
    out = C.c_int()
    rc = lib().or_kadabra_check(d.ctypes.data_as(C.POINTER(C.c_uint64)), d.shape[0], num, omega, eps, delta_v,
                                C.byref(out))
    if rc:
        raise OracleError(rc, "domain")
    return bool(out.value)


def sample_frames(g: Graph, seed: int, spf: int, first: int, count: int, threads: int = 1) -> list[np.ndarray]:
    lab, _ = components(g)
    if threads > 1:
        lens = np.zeros(max(count, 1), np.uint64)
        u32, u64 = C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)
        fn = lib().or_sample_frames_threads
        fn.argtypes = [C.POINTER(_Graph), u32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, u64, u32,
                       C.c_uint64]
        fn.restype = C.c_uint64
        cap = max(1024, count * 64)
        ids = np.empty(cap, np.uint32)
        total = fn(C.byref(g._g), lab.ctypes.data_as(u32), seed, spf, first, count, threads, lens.ctypes.data_as(u64),
                   ids.ctypes.data_as(u32), cap)
        if total > cap:  # rerun with room for every increment
            cap = int(total)
            ids = np.empty(cap, np.uint32)
            fn(C.byref(g._g), lab.ctypes.data_as(u32), seed, spf, first, count, threads, lens.ctypes.data_as(u64),
               ids.ctypes.data_as(u32), cap)
        bounds = np.concatenate([[0], np.cumsum(lens[:count])]).astype(np.int64)
        return [ids[bounds[i]:bounds[i + 1]].copy() for i in range(count)]
    sc = lib().or_scratch_new(g.n)
    out = []
    cap = max(1024, g.n * 4)
    buf = np.empty(cap, np.uint32)
    try:
        for p in range(first, first + count):
            k = lib().or_sample_frame(C.byref(g._g), lab.ctypes.data_as(C.POINTER(C.c_uint32)), seed, p, spf,
                                      buf.ctypes.data_as(C.POINTER(C.c_uint32)), cap, sc)
            if k > cap:
                cap = int(k)
                buf = np.empty(cap, np.uint32)
                k = lib().or_sample_frame(C.byref(g._g), lab.ctypes.data_as(C.POINTER(C.c_uint32)), seed, p, spf,
                                          buf.ctypes.data_as(C.POINTER(C.c_uint32)), cap, sc)
            out.append(buf[:k].copy())
    finally:
        lib().or_scratch_free(sc)
    return out


@dataclass
class Result:
    tau: int
    check_cycles: int
    stop_epoch: int
    omega: int
    diameter_bound: int
    reason: str
    edges_scanned: int
    vertices_expanded: int
    counts: np.ndarray
    scores: np.ndarray
    degenerate_steps: int = 0


def estimate_bc(g: Graph, eps: float, delta: float, *, mode: int = MODE_INDEXED, spf: int = 1,
                epoch_samples: int = 1, seed: int = 1, nominal_threads: int = 1, max_frames: int = 0,
                threads: int = 1) -> Result:
    """threads > 1: frames sampled in parallel and folded in position order
    (or_estimate_bc_threads); results identical to threads = 1."""
    cfg = _Config(mode, nominal_threads, spf, epoch_samples, seed, max_frames, 0.5)
    counts = np.empty(max(g.n, 1), np.uint64)
    scores = np.empty(max(g.n, 1), np.float64)
    res = _Result()
    err = C.create_string_buffer(256)
    fn = lib().or_estimate_bc
    extra = ()
    if threads > 1:
        fn, extra = lib().or_estimate_bc_threads, (threads,)
    rc = fn(C.byref(g._g), eps, delta, C.byref(cfg), *extra, counts.ctypes.data_as(C.POINTER(C.c_uint64)),
                              scores.ctypes.data_as(C.POINTER(C.c_double)), C.byref(res), err, 256)
    if rc:
        raise OracleError(rc, err.value.decode())
    return Result(res.tau, res.check_cycles, res.stop_epoch, res.omega, res.diameter_bound, REASONS[res.reason],
                  res.edges_scanned, res.vertices_expanded, counts[: g.n], scores[: g.n], res.degenerate_steps)


def brandes(g: Graph, threads: int | None = None) -> np.ndarray:
    bc = np.empty(max(g.n, 1), np.float64)
    lib().or_brandes(C.byref(g._g), bc.ctypes.data_as(C.POINTER(C.c_double)), threads or os.cpu_count() or 1)
    return bc[: g.n]


GEN_KINDS = {"gnm": 0, "rmat": 1, "ba": 2, "grid": 3}


def gen_pairs(kind: str, params, lcc: bool = True) -> np.ndarray:
    """The benchmark graphs from gen.c (independent of libadsb.so; equal to
    paper_1903_09422_b200.datasets' generators, tests/test_oracle.py)."""
    L = lib()
    fn = L.or_gen_pairs
    fn.argtypes = [C.c_int, C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_uint64)]
    fn.restype = C.POINTER(C.c_uint64)
    L.or_free.argtypes = [C.c_void_p]
    L.or_free.restype = None
    par = (C.c_double * 8)(*[float(x) for x in params])
    m = C.c_uint64()
    ptr = fn(GEN_KINDS[kind], par, int(lcc), C.byref(m))
    if not ptr:
        return np.zeros(0, np.uint64)
    out = np.ctypeslib.as_array(ptr, shape=(2 * m.value,)).copy() if m.value else np.zeros(0, np.uint64)
    L.or_free(C.cast(ptr, C.c_void_p))
    return out


def write_dense_edges(path, pairs: np.ndarray) -> None:
    """u32 n, u64 m, m x (u32, u32) first-appearance dense ids (ref_driver --graph-bin)."""
    a = np.ascontiguousarray(pairs, dtype=np.uint64)
    fn = lib().or_write_dense_edges
    fn.argtypes = [C.c_char_p, C.POINTER(C.c_uint64), C.c_uint64]
    if fn(os.fsencode(str(path)), a.ctypes.data_as(C.POINTER(C.c_uint64)), a.shape[0] // 2):
        raise OracleError(1, f"cannot write {path}")


def fnv1a(counts: np.ndarray) -> str:
    """FNV-1a 64 over the little-endian u64 counts (ref_driver.cpp:fnv1a)."""
    h = 0xcbf29ce484222325
    for byte in np.ascontiguousarray(counts, dtype="<u8").tobytes():
        h ^= byte
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


# ---------------------------------------------------------------- compiled reference
def ref_available() -> bool:
    return REF_DRIVER.exists()


def ref_run(graph_path, *, eps: float, delta: float, seed: int, variant: str = "indexed", spf: int = 1,
            threads: int = 1, check_interval: int = 1000, max_cycles: int = 0, counts_path=None,
            timeout: float | None = None, reps: int = 1, graph_flag: str = "--graph") -> dict:
    cmd = [str(REF_DRIVER), "run", graph_flag, str(graph_path), "--eps", repr(eps), "--delta", repr(delta),
           "--seed", str(seed), "--variant", variant, "--spf", str(spf), "--threads", str(threads),
           "--check-interval", str(check_interval), "--max-cycles", str(max_cycles), "--reps", str(reps)]
    if counts_path:
        cmd += ["--counts", str(counts_path)]
    out = subprocess.run(cmd, capture_output=True, text=True, check=True, timeout=timeout)
    return json.loads(out.stdout)


def ref_run_bin(graph_path, **kw) -> dict:
    """ref_run on a dense-pairs file (write_dense_edges), ingested by Graph::from_edges."""
    return ref_run(graph_path, graph_flag="--graph-bin", **kw)


def ref_frames(graph_path, *, seed: int, spf: int, first: int, count: int, out_path) -> list[np.ndarray]:
    subprocess.run([str(REF_DRIVER), "frames", "--graph", str(graph_path), "--seed", str(seed), "--spf", str(spf),
                    "--first", str(first), "--count", str(count), "--out", str(out_path)], check=True)
    raw = Path(out_path).read_bytes()
    frames, pos = [], 0
    for _ in range(count):
        (k,) = np.frombuffer(raw, dtype="<u8", count=1, offset=pos)
        pos += 8
        frames.append(np.frombuffer(raw, dtype="<u4", count=int(k), offset=pos).copy())
        pos += 4 * int(k)
    return frames


def ref_dub(graph_path) -> dict:
    out = subprocess.run([str(REF_DRIVER), "dub", "--graph", str(graph_path)], capture_output=True, text=True,
                         check=True)
    return json.loads(out.stdout)

"""Python mirror of `adsamp::kadabra` (kadabra.hpp), backed by libadsb.so.

estimate_bc (kadabra.hpp:308-348) runs the whole pipeline on the GPU:
components and the diameter bound (device kernels), omega (host, libm), then
the deterministic frame pipeline for `indexed`/`sequential` or the cumulative
epoch pipeline for `barrier`/`local`/`shared`.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from ._lib import DomainError, InvalidArgument, Stats, check, dblp, lib, u32p, u64p
from .adsamp import EngineConfig, Graph, QueueStats, RunResult, Variant


def allocate_deltas(n: int, delta: float) -> tuple[np.ndarray, np.ndarray]:
    """kadabra.hpp:30-36"""
    if not (0.0 < delta < 1.0):
        raise InvalidArgument("delta must lie in (0,1)")
    each = delta / (2.0 * float(n))
    return np.full(n, each), np.full(n, each)


def compute_omega(diameter_bound: int, epsilon: float, delta: float, c: float = 0.5) -> int:
    """kadabra.hpp:41-53"""
    out = C.c_uint64()
    check(lib().adsb_compute_omega(diameter_bound, epsilon, delta, c, C.byref(out)))
    return out.value


def f_bound(b_tilde: float, delta_l: float, omega: int, tau: int) -> float:
    """kadabra.hpp:80-84"""
    out = C.c_double()
    check(lib().adsb_f_bound(b_tilde, delta_l, omega, tau, C.byref(out)))
    return out.value


def g_bound(b_tilde: float, delta_u: float, omega: int, tau: int) -> float:
    """kadabra.hpp:87-91"""
    out = C.c_double()
    check(lib().adsb_g_bound(b_tilde, delta_u, omega, tau, C.byref(out)))
    return out.value


def kadabra_check(data, num: int, omega: int, epsilon: float, delta: float) -> bool:
    """kadabra.hpp:148-151 on a host count vector with uniform deltas delta/(2n)."""
    d = np.ascontiguousarray(np.asarray(data, dtype=np.uint64))
    out = C.c_int()
    check(lib().adsb_kadabra_check(d.ctypes.data_as(u64p), d.shape[0], num, omega, epsilon, delta, C.byref(out)))
    return bool(out.value)


class StopReason(enum.IntEnum):
    """kadabra.hpp:289 (+ `capped` for max_cycles runs)"""
    eps_converged = 0
    omega_reached = 1
    capped = 2


def to_string(r: StopReason) -> str:
    return StopReason(r).name


@dataclass
class BcResult:
    """kadabra.hpp:295-304, plus the device counters of the executed sampler.

    `scores` (data[v] / tau, kadabra.hpp:334-337) are filled by the C ABI in
    the estimate_bc call itself, as the reference returns them."""
    _scores: np.ndarray | None = field(default=None, repr=False)
    tau: int = 0
    reason: StopReason = StopReason.eps_converged
    omega: int = 0
    diameter_bound: int = 0
    preprocess_seconds: float = 0.0
    ads_seconds: float = 0.0
    run: RunResult = field(default_factory=lambda: RunResult(np.zeros(0, np.uint64)))
    num_components: int = 0
    edges_scanned: int = 0
    vertices_expanded: int = 0
    kernel_launches: int = 0
    sampler_ms: float = 0.0
    rebuild_edges: int = 0
    backtrack_edges: int = 0
    store_fallbacks: int = 0
    degenerate_steps: int = 0
    world: int = 1

    @property
    def scores(self) -> np.ndarray:
        return self._scores if self._scores is not None else np.zeros(len(self.run.data), dtype=np.float64)


def estimate_bc(g: Graph, epsilon: float, delta: float, config: EngineConfig | None = None,
                audit=None) -> BcResult:
    """kadabra.hpp:308-348. `audit` (AuditSink) is accepted for signature parity; the
    device pipeline has no per-thread event log (out of scope)."""
    cfg = config or EngineConfig()
    cfg.validate()
    n = g.num_vertices()
    counts = np.empty(max(n, 1), dtype=np.uint64)
    scores = np.empty(max(n, 1), dtype=np.float64)
    st = Stats()
    c = cfg.to_c()
    check(lib().adsb_estimate_bc(g.handle, epsilon, delta, C.byref(c), scores.ctypes.data_as(dblp),
                                 counts.ctypes.data_as(u64p), C.byref(st)))
    run = RunResult(data=counts[:n], num=st.tau, total_samples=st.total_samples,
                    per_thread_samples=[st.total_samples], check_cycles=st.check_cycles,
                    stop_epoch=st.stop_epoch,
                    queue=QueueStats(st.queue_max_depth, st.queue_mean_depth, st.queue_allocated,
                                     bool(st.queue_high_water_exceeded)))
    return BcResult(_scores=scores[:n], tau=st.tau, reason=StopReason(st.reason), omega=st.omega,
                    diameter_bound=st.diameter_bound, preprocess_seconds=st.preprocess_seconds,
                    ads_seconds=st.ads_seconds, run=run, num_components=st.num_components,
                    edges_scanned=st.edges_scanned, vertices_expanded=st.vertices_expanded,
                    kernel_launches=st.kernel_launches, sampler_ms=st.sampler_ms,
                    rebuild_edges=st.rebuild_edges, backtrack_edges=st.backtrack_edges,
                    store_fallbacks=st.store_fallbacks, degenerate_steps=st.degenerate_steps,
                    world=st.world)


def sample_frames(g: Graph, seed: int, samples_per_frame: int, first: int, count: int,
                  device: int = -1) -> list[np.ndarray]:
    """Interior vertices of frames [first, first+count) exactly as run_indexed draws them
    (engine.hpp:595-610 keying, kadabra.hpp:250-258 sampling), each sample t->s."""
    offsets = np.empty(count + 1, dtype=np.uint64)
    cap = 0
    incs = np.empty(1, dtype=np.uint32)
    for _ in range(2):
        check(lib().adsb_sample_frames(g.handle, device, seed, samples_per_frame, first, count,
                                       offsets.ctypes.data_as(u64p), incs.ctypes.data_as(u32p), cap))
        need = int(offsets[-1]) if count else 0
        if need <= cap:
            break
        cap = need
        incs = np.empty(max(cap, 1), dtype=np.uint32)
    return [incs[int(offsets[i]):int(offsets[i + 1])].copy() for i in range(count)]


def exact_bc(g: Graph, device: int = -1) -> tuple[np.ndarray, float]:
    """Exact betweenness of every vertex on the device (Brandes, f64), normalised by
    n(n-1) like BcResult::scores; the validation the reference runs with ApspOracle
    (tests/test_util.hpp:164-206). Returns (scores, kernel milliseconds)."""
    n = g.num_vertices()
    out = np.zeros(n, dtype=np.float64)
    ms = C.c_double(0.0)
    check(lib().adsb_exact_bc(g.handle, device, out.ctypes.data_as(dblp), C.byref(ms)))
    return out, ms.value


__all__ = ["allocate_deltas", "compute_omega", "f_bound", "g_bound", "kadabra_check", "StopReason",
           "to_string", "BcResult", "estimate_bc", "exact_bc", "sample_frames", "Variant"]

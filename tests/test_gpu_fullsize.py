"""GPU parity at BASELINE.json sizes and against exact betweenness.

The oracle finishes only small cases in seconds, so the full-size configs are
checked through size-independent properties:

* exact BC on the device (Brandes, f64; kadabra.exact_bc) first agrees with the
  oracle's Brandes (oracle.c or_brandes) to rounding on small graphs;
* the (eps, delta) guarantee: every estimate within eps of exact BC on an
  R-MAT graph of C2's shape (scale 16), deterministic and cumulative-epoch
  modes (tolerance = eps, written in the test);
* C2 at full size: the cumulative-epoch (non-det) estimate within eps of the
  deterministic (indexed-frame) estimate, which is the reference's own output
  (bit-exact against the oracle / compiled reference on every smaller graph);
* C3 at full size: the deterministic result is the same with every sampler
  store (shared-memory table, global state, 128-thread blocks), and its first
  frames equal the oracle's;
* a deep, low-degree lattice with holes (C4's shape, smaller): sampled paths
  equal the oracle's on the global-state store with thread-per-vertex
  expansion; C4 itself: a capped full-size run equals the oracle's counts,
  and test_gpu_parity.py::test_degenerate_sigma_frames_c4 pins the
  all-sigma-wrapped backtrack step;
* C5 at full size: paths identical with and without the shared-memory table,
  and the fused epoch run reproducible run to run.
"""
import numpy as np
import pytest

import oracle
from paper_1903_09422_b200 import adsamp, datasets
from paper_1903_09422_b200.adsamp import EngineConfig, Variant
from paper_1903_09422_b200.kadabra import estimate_bc, exact_bc, sample_frames

from conftest import SMALL_GRAPHS

pytestmark = pytest.mark.gpu


def both(pairs):
    return adsamp.graph_from_pairs(pairs), oracle.from_pairs(pairs)


RMAT = dict(a=0.57, b=0.19, c=0.19)


@pytest.mark.parametrize("name", ["path3", "star4", "cycle4", "cube", "k23", "er100", "two_components", "c1", "rmat11"])
def test_exact_bc_matches_oracle_brandes(name):
    if name == "c1":
        pairs = datasets.pairs("c1_er")
    elif name == "rmat11":
        pairs = datasets.gen_rmat(11, 16, RMAT["a"], RMAT["b"], RMAT["c"], 5)
    else:
        pairs = SMALL_GRAPHS[name]()
    pg, og = both(pairs)
    got, ms = exact_bc(pg.graph, device=0)
    want = oracle.brandes(og)
    assert ms >= 0.0
    np.testing.assert_allclose(got, want, rtol=1e-9, atol=1e-15)


@pytest.fixture(scope="module")
def rmat16():
    pairs = datasets.gen_rmat(16, 16, RMAT["a"], RMAT["b"], RMAT["c"], 16)
    pg = adsamp.graph_from_pairs(pairs)
    exact, _ = exact_bc(pg.graph, device=0)
    return pg, exact


@pytest.mark.parametrize("variant", [Variant.indexed, Variant.shared])
def test_estimates_within_eps_of_exact_rmat16(rmat16, variant):
    pg, exact = rmat16
    eps = 0.005
    cfg = EngineConfig(variant=variant, samples_per_frame=1, threads=8, base_seed=42, device=0)
    r = estimate_bc(pg.graph, eps, 0.1, cfg)
    assert r.reason.name == "eps_converged"
    err = np.max(np.abs(r.scores - exact))
    assert err <= eps, f"max |estimate - exact| = {err} > eps = {eps}"


def test_c2_fullsize_nondet_within_eps_of_deterministic():
    w = datasets.CONFIGS["c2_rmat18"]
    g = datasets.graph("c2_rmat18").graph
    det = estimate_bc(g, w.epsilon, w.delta,
                      EngineConfig(variant=Variant.indexed, samples_per_frame=1, threads=8, base_seed=42, device=0))
    nd = estimate_bc(g, w.epsilon, w.delta,
                     EngineConfig(variant=Variant.shared, threads=8, base_seed=42, device=0))
    nd2 = estimate_bc(g, w.epsilon, w.delta,
                      EngineConfig(variant=Variant.shared, threads=8, base_seed=42, device=0))
    # epochs are index ranges: the non-det mode is reproducible run to run
    assert nd.tau == nd2.tau
    np.testing.assert_array_equal(nd.run.data, nd2.run.data)
    assert det.reason.name == nd.reason.name == "eps_converged"
    assert np.max(np.abs(nd.scores - det.scores)) <= w.epsilon
    # every sample credits d(s,t)-1 interior vertices: counts are bounded by tau each
    assert int(nd.run.data.max()) <= nd.tau and int(det.run.data.max()) <= det.tau


@pytest.mark.parametrize("mode", ["block-global", "block-128"])
def test_c3_fullsize_deterministic_store_invariance(mode, monkeypatch):
    w = datasets.CONFIGS["c3_ba"]
    pairs = datasets.pairs("c3_ba")
    cfg = EngineConfig(variant=Variant.indexed, samples_per_frame=1, threads=8, base_seed=w.seed, device=0)
    monkeypatch.setenv("ADSB_SAMPLER", "block")
    monkeypatch.delenv("ADSB_NO_SMEM", raising=False)
    monkeypatch.delenv("ADSB_BLOCK", raising=False)
    ref = estimate_bc(adsamp.graph_from_pairs(pairs).graph, w.epsilon, w.delta, cfg)
    if mode == "block-global":
        monkeypatch.setenv("ADSB_NO_SMEM", "1")
    else:
        monkeypatch.setenv("ADSB_BLOCK", "128")
    got = estimate_bc(adsamp.graph_from_pairs(pairs).graph, w.epsilon, w.delta, cfg)
    assert (got.tau, got.run.check_cycles, got.reason.name) == (ref.tau, ref.run.check_cycles, ref.reason.name)
    np.testing.assert_array_equal(got.run.data, ref.run.data)


def test_c3_fullsize_first_frames_match_oracle():
    pairs = datasets.pairs("c3_ba")
    pg, og = both(pairs)
    got = sample_frames(pg.graph, 42, 1, 0, 24, device=0)
    want = oracle.sample_frames(og, 42, 1, 0, 24)
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("mode", ["global", "auto"])
def test_holey_lattice_lowdegree_frames(mode, monkeypatch):
    monkeypatch.setenv("ADSB_SAMPLER", "block")
    if mode == "global":
        monkeypatch.setenv("ADSB_NO_SMEM", "1")
    else:
        monkeypatch.delenv("ADSB_NO_SMEM", raising=False)
    pairs = datasets.gen_grid(300, 300, 0.1, 5)
    pg, og = both(pairs)
    got = sample_frames(pg.graph, 11, 2, 3, 60, device=0)
    want = oracle.sample_frames(og, 11, 2, 3, 60)
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a, b)
    cfg = EngineConfig(variant=Variant.indexed, samples_per_frame=1, threads=8, base_seed=11, max_cycles=500, device=0)
    r = estimate_bc(pg.graph, 0.02, 0.1, cfg)
    o = oracle.estimate_bc(og, 0.02, 0.1, spf=1, seed=11, nominal_threads=8, max_frames=500)
    assert (r.tau, r.run.check_cycles) == (o.tau, o.check_cycles)
    np.testing.assert_array_equal(r.run.data, o.counts)


@pytest.fixture(scope="module")
def c5_csr():
    g = datasets.graph("c5_rmat24").graph
    return g.num_vertices(), np.ascontiguousarray(g.offsets()), np.ascontiguousarray(g.neighbor_list())


def test_c5_fullsize_store_invariance_and_reproducibility(c5_csr, monkeypatch):
    """C5 at full size (8.9M vertices, 2.1 GB CSR): sampled paths are the same
    with the shared-memory table (+ global fallback with the membership filter)
    and with the global store alone; the fused cumulative-epoch run is
    reproducible run to run (epochs are index ranges)."""
    n, off, nb = c5_csr
    monkeypatch.setenv("ADSB_SAMPLER", "block")
    monkeypatch.delenv("ADSB_NO_SMEM", raising=False)
    g1 = adsamp.Graph.from_csr(n, off, nb)
    a = sample_frames(g1, 42, 1, 0, 400, device=0)
    monkeypatch.setenv("ADSB_NO_SMEM", "1")
    g2 = adsamp.Graph.from_csr(n, off, nb)
    b = sample_frames(g2, 42, 1, 0, 400, device=0)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    assert sum(len(x) for x in a) > 400
    monkeypatch.delenv("ADSB_NO_SMEM", raising=False)
    w = datasets.CONFIGS["c5_rmat24"]
    cfg = EngineConfig(variant=Variant.shared, threads=8, base_seed=42, device=0, max_cycles=48)
    r1 = estimate_bc(g1, w.epsilon, w.delta, cfg)
    r2 = estimate_bc(g1, w.epsilon, w.delta, cfg)
    assert r1.tau == r2.tau == 48 * 1024 and r1.reason.name == "capped"
    np.testing.assert_array_equal(r1.run.data, r2.run.data)


def test_c4_fullsize_capped_run_matches_oracle():
    """C4 at full size (2048^2 lattice with holes, 4.19M vertices, sigma wraps
    mod 2^64): a capped deterministic run on the global store (cleared layout,
    512-thread teams, batched claims, push rebuild) gives the oracle's tau and
    every per-vertex count."""
    pairs = datasets.pairs("c4_grid")
    pg, og = both(pairs)
    cfg = EngineConfig(variant=Variant.indexed, samples_per_frame=1, threads=8, base_seed=42, max_cycles=24, device=0)
    r = estimate_bc(pg.graph, 0.01, 0.1, cfg)
    o = oracle.estimate_bc(og, 0.01, 0.1, spf=1, seed=42, nominal_threads=8, max_frames=24)
    assert (r.tau, r.run.check_cycles, r.reason.name) == (o.tau, o.check_cycles, o.reason) == (24, 24, "capped")
    np.testing.assert_array_equal(r.run.data, o.counts)
    assert int(r.run.data.sum()) > 24 * 500  # deep paths: hundreds of interior vertices each


# ----------------------------------------------------------------------------- full-size goldens
# tests/golden/fullsize.json (tests/golden/make_fullsize.py): the compiled
# reference's run_indexed on C2 and C3 (equal to the threaded oracle), the
# threaded oracle's runs on C4 (where the reference segfaults) and C2's
# cumulative epochs, C5's first 200 frames, and n/m/components/D_ub/omega of
# every config. Each graph is regenerated here and pinned by its pairs hash.
import hashlib  # noqa: E402
import json  # noqa: E402
from pathlib import Path  # noqa: E402

FULL = json.loads((Path(__file__).resolve().parent / "golden" / "fullsize.json").read_text())


def _pairs_sha(p) -> str:
    return hashlib.sha256(np.ascontiguousarray(p, dtype="<u8").tobytes()).hexdigest()


@pytest.fixture(scope="module")
def full_graphs():
    cache = {}

    def get(name):
        if name not in cache:
            pairs = datasets.pairs(name)
            if name in FULL["graphs"]:
                assert _pairs_sha(pairs) == FULL["graphs"][name]["pairs_sha256"], f"generator drift for {name}"
            cache.clear()  # one full-size graph resident at a time
            cache[name] = adsamp.graph_from_pairs(pairs).graph
        return cache[name]
    return get


@pytest.mark.parametrize("name", sorted(FULL["graphs"]))
def test_fullsize_graph_facts_match_oracle(full_graphs, name):
    """n, m, components, D_ub (graph.hpp:202-214) and omega (kadabra.hpp:41-53)
    computed on the device equal the oracle's at every config's full size."""
    want = FULL["graphs"][name]
    g = full_graphs(name)
    assert (g.num_vertices(), g.num_edges()) == (want["n"], want["m"])
    cc = adsamp.connected_components(g, device=0)
    assert cc.num_components == want["components"]
    dub = adsamp.diameter_upper_bound(g, device=0)
    assert dub == want["diameter_bound"]
    from paper_1903_09422_b200.kadabra import compute_omega
    assert compute_omega(dub, want["epsilon"], want["delta"]) == want["omega"]


@pytest.mark.parametrize("key", sorted(FULL["runs"]))
def test_fullsize_run_matches_golden(full_graphs, key):
    """The whole run at the config's own size: tau, check cycles, stop epoch,
    reason and the FNV-1a of every per-vertex count equal the reference's
    indexed-frame run (C2, C3) or the oracle's (C4, C2 epochs)."""
    want = FULL["runs"][key]
    g = full_graphs(want["config"])
    if want["mode"] == "indexed":
        cfg = EngineConfig(variant=Variant.indexed, samples_per_frame=want["spf"], threads=want["nominal_threads"],
                           base_seed=want["seed"], device=0)
    else:
        cfg = EngineConfig(variant=Variant.shared, epoch_samples=want["epoch_samples"], threads=8,
                           base_seed=want["seed"], device=0)
    r = estimate_bc(g, want["epsilon"], want["delta"], cfg)
    got = (r.tau, r.run.check_cycles, r.run.stop_epoch, r.reason.name, r.omega, r.diameter_bound,
           oracle.fnv1a(r.run.data), int(r.run.data.sum()), int(r.run.data.max()))
    exp = (want["tau"], want["check_cycles"], want["stop_epoch"], want["reason"], want["omega"],
           want["diameter_bound"], want["counts_fnv1a"], want["counts_sum"], want["counts_max"])
    assert got == exp, (key, got, exp)
    # the device counts all-sigma-wrapped backtrack steps over every sample it
    # drew (including those past the stop, which are discarded); the oracle
    # over the tau consumed ones
    assert r.degenerate_steps >= want["degenerate_steps"]
    assert (r.degenerate_steps == 0) == (want["degenerate_steps"] == 0)


def _fnv1a_u32(ids: np.ndarray) -> str:
    h = 0xcbf29ce484222325
    for byte in np.ascontiguousarray(ids, dtype="<u4").tobytes():
        h ^= byte
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


@pytest.mark.parametrize("key", sorted(FULL["frames"]))
def test_fullsize_frames_match_golden(full_graphs, key):
    """C5 (R-MAT 24, 8.9M vertices): the first 200 frames' sampled paths — the
    RNG stream and every sigma-weighted backtrack choice — equal the oracle's."""
    want = FULL["frames"][key]
    g = full_graphs(want["config"])
    got = sample_frames(g, want["seed"], want["spf"], want["first"], want["count"], device=0)
    assert [len(x) for x in got] == want["lens"]
    ids = np.concatenate(got) if got else np.zeros(0, np.uint32)
    assert _fnv1a_u32(ids) == want["ids_fnv1a"]


def test_c5_nondet_within_2eps_of_deterministic(full_graphs):
    """the reference's own C5 output is infeasible (~10^7
    core-seconds), so the non-deterministic estimate is checked against the
    deterministic (indexed-frame) mode, which is bit-exact against the
    reference wherever the reference finishes. Both estimate BC within eps
    with probability >= 1 - delta, so the sound tolerance between them is 2 eps."""
    w = datasets.CONFIGS["c5_rmat24"]
    g = full_graphs("c5_rmat24")
    det = estimate_bc(g, w.epsilon, w.delta,
                      EngineConfig(variant=Variant.indexed, samples_per_frame=1, threads=8, base_seed=42, device=0))
    nd = estimate_bc(g, w.epsilon, w.delta, EngineConfig(variant=Variant.shared, threads=8, base_seed=42, device=0))
    assert det.reason.name == nd.reason.name == "eps_converged"
    err = float(np.max(np.abs(nd.scores - det.scores)))
    assert err <= 2 * w.epsilon, f"max |nondet - det| = {err} > 2 eps"

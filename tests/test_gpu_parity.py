"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bit-exact for all integer outputs: sampled paths (and therefore RNG stream
consumption), per-vertex counts, tau, check_cycles, stop_epoch, D_ub, omega,
component labels. The oracle itself is pinned to the compiled reference in
tests/test_oracle.py and tests/golden/.
"""
import numpy as np
import pytest

import oracle
from paper_1903_09422_b200 import adsamp, datasets, kadabra
from paper_1903_09422_b200.adsamp import EngineConfig, Variant
from paper_1903_09422_b200.kadabra import estimate_bc, sample_frames

from conftest import SMALL_GRAPHS

pytestmark = pytest.mark.gpu


def both(pairs):
    return adsamp.graph_from_pairs(pairs), oracle.from_pairs(pairs)


@pytest.fixture(scope="module")
def c1():
    p = datasets.pairs("c1_er")
    return both(p)


@pytest.fixture(scope="module")
def grid200():
    # 200x200 lattice with no drops: sigma exceeds 2^64 for most far pairs (wrap parity)
    p = datasets.gen_grid(200, 200, 0.0, 3)
    return both(p)


@pytest.mark.parametrize("name", sorted(SMALL_GRAPHS))
def test_components_and_dub(name):
    pg, og = both(SMALL_GRAPHS[name]())
    cc = adsamp.connected_components(pg.graph)
    lab, comps = oracle.components(og)
    assert cc.num_components == comps
    np.testing.assert_array_equal(cc.label, lab)
    assert adsamp.diameter_upper_bound(pg.graph) == oracle.diameter_upper_bound(og)
    for s in range(min(og.n, 5)):
        assert adsamp.eccentricity(pg.graph, s) == oracle.eccentricity(og, s)


def test_components_labels_stable_over_many_builds():
    """Regression: union-find path halving once raced with uf_compress and
    mislabelled about one vertex in a thousand builds (samples touching it were
    dropped as disconnected pairs). Fresh handles recompute the labels."""
    cases = [datasets.pairs("c1_er"), datasets.gen_gnm(6000, 4000, 5, lcc=False)]  # connected; many components
    for pairs in cases:
        lab, comps = oracle.components(oracle.from_pairs(pairs))
        for _ in range(150):
            cc = adsamp.connected_components(adsamp.graph_from_pairs(pairs).graph)
            assert cc.num_components == comps
            np.testing.assert_array_equal(cc.label, lab)


@pytest.mark.parametrize("name", sorted(SMALL_GRAPHS))
@pytest.mark.parametrize("spf", [1, 3])
def test_frames_small(name, spf):
    pg, og = both(SMALL_GRAPHS[name]())
    got = sample_frames(pg.graph, 1234, spf, 0, 200)
    want = oracle.sample_frames(og, 1234, spf, 0, 200)
    for p, (a, b) in enumerate(zip(got, want)):
        np.testing.assert_array_equal(a, b, err_msg=f"frame {p}")


def test_frames_c1(c1):
    pg, og = c1
    got = sample_frames(pg.graph, 42, 1, 0, 4000)
    want = oracle.sample_frames(og, 42, 1, 0, 4000)
    assert sum(len(x) for x in want) > 4000
    for p, (a, b) in enumerate(zip(got, want)):
        np.testing.assert_array_equal(a, b, err_msg=f"frame {p}")
    got = sample_frames(pg.graph, 42, 1000, 7, 3)
    want = oracle.sample_frames(og, 42, 1000, 7, 3)
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a, b)


def test_frames_sigma_wrap(grid200):
    pg, og = grid200
    got = sample_frames(pg.graph, 9, 2, 100, 60)
    want = oracle.sample_frames(og, 9, 2, 100, 60)
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("name", ["path3", "star4", "cycle4", "cube", "k23", "er100", "two_components"])
@pytest.mark.parametrize("spf", [1, 7])
def test_estimate_det_small(name, spf):
    pg, og = both(SMALL_GRAPHS[name]())
    cfg = EngineConfig(variant=Variant.indexed, samples_per_frame=spf, base_seed=5, threads=4)
    r = estimate_bc(pg.graph, 0.05, 0.1, cfg)
    o = oracle.estimate_bc(og, 0.05, 0.1, spf=spf, seed=5, nominal_threads=4)
    assert (r.tau, r.run.check_cycles, r.run.stop_epoch, r.omega, r.diameter_bound) == \
           (o.tau, o.check_cycles, o.stop_epoch, o.omega, o.diameter_bound)
    assert r.reason.name == o.reason
    np.testing.assert_array_equal(r.run.data, o.counts)
    np.testing.assert_array_equal(r.scores, o.scores)


@pytest.mark.parametrize("spf", [1, 1000])
def test_estimate_det_c1(c1, spf):
    pg, og = c1
    cfg = EngineConfig(variant=Variant.indexed, samples_per_frame=spf, base_seed=42, threads=8)
    r = estimate_bc(pg.graph, 0.01, 0.1, cfg)
    o = oracle.estimate_bc(og, 0.01, 0.1, spf=spf, seed=42, nominal_threads=8)
    assert (r.tau, r.run.check_cycles, r.run.stop_epoch) == (o.tau, o.check_cycles, o.stop_epoch)
    assert r.reason.name == o.reason == "eps_converged"
    np.testing.assert_array_equal(r.run.data, o.counts)
    assert r.run.total_samples >= r.tau


@pytest.mark.parametrize("B", [64, 1000])
def test_estimate_epoch_small(B):
    pg, og = both(SMALL_GRAPHS["er100"]())
    cfg = EngineConfig(variant=Variant.shared, threads=4, base_seed=11, epoch_samples=B)
    r = estimate_bc(pg.graph, 0.05, 0.1, cfg)
    o = oracle.estimate_bc(og, 0.05, 0.1, mode=oracle.MODE_EPOCH, epoch_samples=B, seed=11)
    assert (r.tau, r.run.check_cycles) == (o.tau, o.check_cycles)
    np.testing.assert_array_equal(r.run.data, o.counts)


def test_estimate_epoch_c1_within_eps_of_brandes(c1):
    pg, og = c1
    exact = oracle.brandes(og)
    cfg = EngineConfig(variant=Variant.shared, threads=8, base_seed=42, epoch_samples=2048)
    r = estimate_bc(pg.graph, 0.01, 0.1, cfg)
    o = oracle.estimate_bc(og, 0.01, 0.1, mode=oracle.MODE_EPOCH, epoch_samples=2048, seed=42)
    np.testing.assert_array_equal(r.run.data, o.counts)  # epoch semantics are reproducible too
    assert np.max(np.abs(r.scores - exact)) <= 0.01      # the (eps, delta) guarantee, eps = 0.01


def test_capped_runs(c1):
    pg, og = c1
    cfg = EngineConfig(variant=Variant.indexed, samples_per_frame=1, base_seed=3, max_cycles=777)
    r = estimate_bc(pg.graph, 0.01, 0.1, cfg)
    o = oracle.estimate_bc(og, 0.01, 0.1, spf=1, seed=3, max_frames=777)
    assert r.tau == o.tau == 777 and r.reason.name == o.reason == "capped"
    np.testing.assert_array_equal(r.run.data, o.counts)


def test_single_vertex_and_errors():
    pg = adsamp.parse_edge_list("7 7\n")
    assert pg.graph.num_vertices() == 1
    r = estimate_bc(pg.graph, 0.05, 0.1, EngineConfig(variant=Variant.indexed))
    assert r.tau == 0 and list(r.scores) == [0.0]
    g = adsamp.Graph.from_edges(3, [(0, 1), (1, 2)])
    with pytest.raises(ValueError):
        estimate_bc(g, 1.5, 0.1, EngineConfig())
    with pytest.raises(ValueError):
        estimate_bc(g, 0.1, 0.0, EngineConfig())


@pytest.mark.parametrize("mode", ["block", "block-vec4", "block-global", "block-tinyhash", "warp"])
def test_sampler_variants_bit_exact(mode, monkeypatch, grid200):
    """All sampler implementations (block teams with the shared-memory table,
    with scalar or 16-byte vector adjacency reads, block teams forced onto
    global state, a table so small that most samples overflow and are redone,
    warp teams) give the same paths and results."""
    monkeypatch.delenv("ADSB_NO_SMEM", raising=False)
    monkeypatch.delenv("ADSB_HASH_CAP", raising=False)
    monkeypatch.setenv("ADSB_VEC4", "1" if mode == "block-vec4" else "0")
    monkeypatch.setenv("ADSB_SAMPLER", "warp" if mode == "warp" else "block")  # small n would pick warps
    if mode == "block-global":
        monkeypatch.setenv("ADSB_NO_SMEM", "1")
    elif mode == "block-tinyhash":
        monkeypatch.setenv("ADSB_HASH_CAP", "64")
    p = datasets.pairs("c1_er")
    pg, og = both(p)  # fresh handle -> fresh device context / arena
    got = sample_frames(pg.graph, 77, 2, 0, 1500)
    want = oracle.sample_frames(og, 77, 2, 0, 1500)
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a, b)
    cfg = EngineConfig(variant=Variant.indexed, samples_per_frame=1, base_seed=42, threads=8)
    r = estimate_bc(pg.graph, 0.01, 0.1, cfg)
    assert r.tau == 10307
    gp = datasets.gen_grid(200, 200, 0.0, 3)
    pg2, og2 = both(gp)
    got = sample_frames(pg2.graph, 9, 1, 0, 40)
    want = oracle.sample_frames(og2, 9, 1, 0, 40)
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a, b)


def test_cpp_dropin_tool_matches_oracle(tmp_path):
    """tools/adsb_run.cpp (written only against include/adsamp_b200.hpp) reproduces
    the reference CLI's score file (adsamp_cli.cpp:99-106 format) bit for bit."""
    import subprocess
    from pathlib import Path
    tool = Path(__file__).resolve().parents[1] / "paper_1903_09422_b200" / "adsb_run"
    path = tmp_path / "c1.edges"
    datasets.write_edge_list(path, datasets.pairs("c1_er"))
    out = tmp_path / "scores.csv"
    res = subprocess.run([str(tool), "--graph", str(path), "--variant", "indexed", "--threads", "8", "--eps", "0.01",
                          "--delta", "0.1", "--seed", "42", "--samples-per-frame", "1", "--output", str(out)],
                         capture_output=True, text=True, check=True)
    assert "tau: 10307  reason: eps_converged" in res.stdout
    og = oracle.parse_file(path)
    o = oracle.estimate_bc(og, 0.01, 0.1, spf=1, seed=42)
    want = "vertex_id,score\n" + "".join("%d,%.10g\n" % (int(i), s) for i, s in zip(og.original_ids, o.scores))
    assert out.read_text() == want


def test_nccl_paths_world1(c1):
    """Exercise the NCCL code paths (epoch all-reduce, deterministic event
    all-gather with sentinel padding and 64-bit sort) with a 1-rank
    communicator: results must equal the communicator-free run."""
    from paper_1903_09422_b200.distributed import Comm
    comm = Comm(1, 0, Comm.unique_id(), 0)
    pg, og = c1
    for variant, extra in [(Variant.indexed, {}), (Variant.shared, {"epoch_samples": 4096})]:
        base = EngineConfig(variant=variant, samples_per_frame=1, base_seed=9, threads=8, **extra)
        with_comm = EngineConfig(variant=variant, samples_per_frame=1, base_seed=9, threads=8, comm=comm, **extra)
        a = estimate_bc(pg.graph, 0.01, 0.1, base)
        b = estimate_bc(pg.graph, 0.01, 0.1, with_comm)
        assert (a.tau, a.run.check_cycles) == (b.tau, b.run.check_cycles)
        np.testing.assert_array_equal(a.run.data, b.run.data)
    comm.close()


def test_degenerate_sigma_frames_c4():
    """On the C4 grid, frame 247 (seed 42) hits a backtrack step where sigma(cur)
    and every predecessor sigma are 0 mod 2^64; the reference's behaviour is
    undefined there (it segfaults). Engine and oracle both take the first
    predecessor in id order, so the paths must still agree."""
    p = datasets.pairs("c4_grid")
    pg, og = both(p)
    got = sample_frames(pg.graph, 42, 1, 244, 6)
    want = oracle.sample_frames(og, 42, 1, 244, 6)
    assert len(want[3]) > 0
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("B", [64, 1024])
def test_epoch_block_teams_fused_and_host_driven(fused, B, monkeypatch):
    """Block-team epoch pipeline, fused (device-side in-order folds + stopping
    rule in one persistent launch) and host-driven (double-buffered epochs on
    two streams): both must equal the oracle's cumulative-epoch restatement."""
    monkeypatch.setenv("ADSB_SAMPLER", "block")
    if not fused:
        monkeypatch.setenv("ADSB_NO_FUSED", "1")
    else:
        monkeypatch.delenv("ADSB_NO_FUSED", raising=False)
    for name, eps in [("er100", 0.05), ("c1", 0.01)]:
        pairs = datasets.pairs("c1_er") if name == "c1" else SMALL_GRAPHS[name]()
        pg, og = both(pairs)
        cfg = EngineConfig(variant=Variant.shared, threads=4, base_seed=13, epoch_samples=B)
        r = estimate_bc(pg.graph, eps, 0.1, cfg)
        o = oracle.estimate_bc(og, eps, 0.1, mode=oracle.MODE_EPOCH, epoch_samples=B, seed=13)
        assert (r.tau, r.run.check_cycles, r.reason.name) == (o.tau, o.check_cycles, o.reason), name
        np.testing.assert_array_equal(r.run.data, o.counts)
        assert r.run.total_samples >= r.tau
    cap = EngineConfig(variant=Variant.shared, threads=4, base_seed=13, epoch_samples=B, max_cycles=3)
    r = estimate_bc(pg.graph, 0.01, 0.1, cap)
    assert r.tau == 3 * B and r.reason.name == "capped"


@pytest.mark.parametrize("mode", ["block", "block-vec4", "block-global", "block-128"])
@pytest.mark.parametrize("spf", [1, 4])
def test_block_teams_frames_ba(mode, spf, monkeypatch):
    """Block teams on a hub-heavy BA graph (shared-memory table overflows for
    some samples and falls back), including spf > 1 (stream continuity across
    samples of one frame)."""
    monkeypatch.setenv("ADSB_SAMPLER", "block")
    monkeypatch.delenv("ADSB_NO_SMEM", raising=False)
    monkeypatch.delenv("ADSB_BLOCK", raising=False)
    monkeypatch.setenv("ADSB_VEC4", "1" if mode == "block-vec4" else "0")
    if mode == "block-global":
        monkeypatch.setenv("ADSB_NO_SMEM", "1")
    elif mode == "block-128":
        monkeypatch.setenv("ADSB_BLOCK", "128")
    p = datasets.gen_ba(1 << 15, 8, 3)
    pg, og = both(p)
    got = sample_frames(pg.graph, 21, spf, 5, 300)
    want = oracle.sample_frames(og, 21, spf, 5, 300)
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a, b)
    cfg = EngineConfig(variant=Variant.indexed, samples_per_frame=spf, base_seed=21, threads=4, max_cycles=600)
    r = estimate_bc(pg.graph, 0.02, 0.1, cfg)
    o = oracle.estimate_bc(og, 0.02, 0.1, spf=spf, seed=21, nominal_threads=4, max_frames=600)
    assert (r.tau, r.run.check_cycles, r.reason.name) == (o.tau, o.check_cycles, o.reason)
    np.testing.assert_array_equal(r.run.data, o.counts)


def test_fused_epoch_audit_replay(tmp_path, monkeypatch):
    """validate_consistency-style replay of the fused epoch pipeline
    (audit.hpp:101-161 analogue): with ADSB_FUSED_AUDIT the
    kernel records, per sample, how many increments it made (and its distance),
    and per epoch how many increments the in-order fold consumed. Every sample
    of a folded epoch must have recorded exactly its path's interior vertices
    (the oracle's path for that stream position), every folded epoch must have
    consumed exactly the sum over its samples, and nothing past the stop epoch
    may be folded."""
    monkeypatch.setenv("ADSB_SAMPLER", "block")
    audit = tmp_path / "audit.bin"
    monkeypatch.setenv("ADSB_FUSED_AUDIT", str(audit))
    pairs = datasets.pairs("c1_er")
    pg, og = both(pairs)
    B = 256
    cfg = EngineConfig(variant=Variant.shared, threads=4, base_seed=5, epoch_samples=B, device=0)
    r = estimate_bc(pg.graph, 0.02, 0.1, cfg)
    a = np.fromfile(audit, dtype=np.uint32)
    max_epochs = a.size // (B + 1)
    per_sample, folded = a[: max_epochs * B], a[max_epochs * B:]
    stop = r.run.check_cycles  # epochs folded, in order
    paths = oracle.sample_frames(og, 5, 1, 0, stop * B)
    rec = per_sample[: stop * B] & 0xFFFF
    np.testing.assert_array_equal(rec, np.array([len(p) for p in paths], dtype=np.uint32))
    np.testing.assert_array_equal(folded[:stop], rec.reshape(stop, B).sum(axis=1))
    assert not folded[stop:].any()
    assert int(folded[:stop].sum()) == int(r.run.data.sum())


def _read_audit(path):
    w = np.fromfile(path, dtype=np.uint64)
    i, recs = 0, []
    while i < w.size:
        kind = int(w[i])
        if kind == 1:
            first, F, cnt, limit, stopped, bm = (int(x) for x in w[i + 1:i + 7])
            i += 7
            run_max = w[i:i + F].astype(np.int64)
            i += F
            ev = w[i:i + cnt]
            i += cnt
            recs.append(("batch", first, F, limit, stopped, bm, run_max, ev))
        elif kind == 2:
            e, B, ok, mx = (int(x) for x in w[i + 1:i + 5])
            i += 5
            recs.append(("round", e, B, ok, mx, w[i:i + recs_n[0]].astype(np.int64)))
            i += recs_n[0]
        elif kind == 3:
            recs.append(("end", int(w[i + 1]), int(w[i + 2])))
            i += 3
        else:
            raise AssertionError(f"bad audit record {kind}")
    return recs


recs_n = [0]


@pytest.mark.parametrize("variant,extra", [(Variant.indexed, {"samples_per_frame": 1}),
                                           (Variant.indexed, {"samples_per_frame": 3}),
                                           (Variant.shared, {"epoch_samples": 256})])
def test_frames_pipeline_audit_replay(tmp_path, monkeypatch, variant, extra):
    """validate_consistency replay (audit.hpp:101-161 analogue) of the frame
    pipeline — the deterministic batches and the multi-rank epoch path (epochs
    as single-sample frames checked every B): every frame's increments equal
    the oracle's path(s) for that stream position, every check record (the
    running max after each frame) equals the max count replayed from the event
    log, the stop frame is the first whose check passes, and the final counts
    are exactly the events of the frames up to it."""
    audit = tmp_path / "audit.bin"
    monkeypatch.setenv("ADSB_AUDIT", str(audit))
    monkeypatch.setenv("ADSB_SAMPLER", "warp")
    pairs = datasets.pairs("c1_er")
    pg, og = both(pairs)
    n = pg.graph.num_vertices()
    eps = 0.03
    cfg = EngineConfig(variant=variant, threads=8, base_seed=9, device=0, **extra)
    r = estimate_bc(pg.graph, eps, 0.1, cfg)
    recs_n[0] = n
    recs = _read_audit(audit)
    spf = extra.get("samples_per_frame", 1)
    C = extra.get("epoch_samples", 1)
    counts = np.zeros(n, np.int64)
    run_max_all = 0
    stop_frame = None
    for rec in recs:
        if rec[0] != "batch":
            continue
        _, first, F, limit, stopped, bm, run_max, ev = rec
        assert bm == run_max_all
        ev = ev[ev != np.uint64(0xFFFFFFFFFFFFFFFF)]
        v = (ev >> np.uint64(32)).astype(np.int64)
        f = (ev & np.uint64(0xFFFFFFFF)).astype(np.int64)
        paths = oracle.sample_frames(og, 9, spf, first, F)
        order = np.argsort(f, kind="stable")
        v, f = v[order], f[order]
        bounds = np.searchsorted(f, np.arange(F + 1))
        cur = counts.copy()
        mx = 0
        for k in range(F):
            got = np.sort(v[bounds[k]:bounds[k + 1]])
            np.testing.assert_array_equal(got, np.sort(paths[k].astype(np.int64)))
            for x in got:
                cur[x] += 1
                mx = max(mx, int(cur[x]))
            assert int(run_max[k]) == mx, (first, k)
        # frames <= limit are folded
        for k in range(limit + 1):
            np.add.at(counts, v[bounds[k]:bounds[k + 1]], 1)
        run_max_all = max(run_max_all, int(run_max[limit]))
        if stopped:
            stop_frame = first + limit
    assert stop_frame is not None
    tau = (stop_frame + 1) * spf
    assert r.tau == tau and recs[-1] == ("end", tau, (stop_frame + 1) // C)
    np.testing.assert_array_equal(r.run.data.astype(np.int64), counts)
    # the stop check holds with the reference's all-vertex rule (kadabra_check)
    assert kadabra.kadabra_check(counts, tau, r.omega, eps, 0.1)


def test_barrier_rounds_audit_replay(tmp_path, monkeypatch):
    """The barrier variant's round pipeline (dense all-reduce of the n-length
    round counts, used across GPUs): every round's counts equal the oracle's
    paths for that round's sample indices, every check's max and verdict are
    reproduced from the running total, and the result is the total at the
    first passing round."""
    audit = tmp_path / "audit.bin"
    monkeypatch.setenv("ADSB_AUDIT", str(audit))
    monkeypatch.setenv("ADSB_DENSE_EPOCHS", "1")
    monkeypatch.setenv("ADSB_NO_FUSED", "1")
    pairs = datasets.pairs("c1_er")
    pg, og = both(pairs)
    n = pg.graph.num_vertices()
    eps, B = 0.03, 500
    cfg = EngineConfig(variant=Variant.barrier, threads=8, base_seed=4, check_interval=B, device=0)
    r = estimate_bc(pg.graph, eps, 0.1, cfg)
    recs_n[0] = n
    recs = [x for x in _read_audit(audit) if x[0] == "round"]
    total = np.zeros(n, np.int64)
    for _, e, B_, ok, mx, cnt in recs:
        assert B_ == B
        want = np.zeros(n, np.int64)
        for p in oracle.sample_frames(og, 4, 1, e * B, B):
            np.add.at(want, p.astype(np.int64), 1)
        np.testing.assert_array_equal(cnt, want)
        total += cnt
        assert mx == int(total.max())
        assert bool(ok) == kadabra.kadabra_check(total, (e + 1) * B, r.omega, eps, 0.1)
        if ok:
            break
    assert r.tau == (recs[-1][1] + 1) * B
    np.testing.assert_array_equal(r.run.data.astype(np.int64), total)


@pytest.mark.parametrize("knobs", [{"ADSB_VEC4": "1"}, {"ADSB_VEC4": "1", "ADSB_HUB_FACTOR": "1"},
                                   {"ADSB_VEC4": "1", "ADSB_NO_HUB_TREES": "1"},
                                   {"ADSB_VEC4": "1", "ADSB_HUB_FACTOR": "1", "ADSB_HASH_CAP": "256"}])
def test_hub_search_trees_match_oracle(knobs, monkeypatch):
    """Hub search trees (hub_index.cuh): in the vector kernels, probe passes and
    backtrack steps by level list find a vertex in a high-degree row through an
    8-ary tree over the row instead of a binary search of it. Sampled paths and
    a whole cumulative-epoch run equal the oracle's with the trees on, with a
    hub threshold that sends far more rows through them, with the trees off,
    and with a tiny table (most samples run on a global region: the fallback
    samples' instantiation of the same searches)."""
    monkeypatch.setenv("ADSB_SAMPLER", "block")
    for k, v in knobs.items():
        monkeypatch.setenv(k, v)
    pairs = datasets.gen_rmat(16, 16, 0.57, 0.19, 0.19, 21)
    pg, og = both(pairs)
    want = oracle.sample_frames(og, 3, 2, 0, 600)
    got = sample_frames(pg.graph, 3, 2, 0, 600, device=0)
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a, b)
    cfg = EngineConfig(variant=Variant.shared, threads=8, base_seed=3, epoch_samples=512, device=0)
    r = estimate_bc(pg.graph, 0.02, 0.1, cfg)
    o = oracle.estimate_bc(og, 0.02, 0.1, mode=oracle.MODE_EPOCH, epoch_samples=512, seed=3)
    assert (r.tau, r.run.check_cycles) == (o.tau, o.check_cycles)
    np.testing.assert_array_equal(r.run.data, o.counts)

"""Pin the CPU oracle (oracle/oracle.c) before trusting it.

1. Known-answer values the reference's own tests hold (test_kadabra.cpp,
   test_engine.cpp, test_graph.cpp, test_util.hpp), restated here.
2. Golden fixtures produced by the compiled reference (tests/golden/, made by
   tests/golden/make_golden.py from oracle/_ref/ref_driver).
3. When the compiled reference is present (this container), live cross-checks
   on freshly generated graphs.
"""
from __future__ import annotations

import json
import math
from decimal import Decimal, getcontext
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_1903_09422_b200 import datasets
from paper_1903_09422_b200.adsamp import SplitMix64, mix64, reseed, stream_rng

from conftest import SMALL_GRAPHS

GOLD = Path(__file__).resolve().parent / "golden"
MASK = (1 << 64) - 1


def golden():
    return json.loads((GOLD / "golden.json").read_text()), np.load(GOLD / "golden_arrays.npz")


# ----------------------------------------------------------------------------- rng.hpp
def test_rng_known_answers():
    # splitmix64 reference vector (seed 0): first outputs of the public algorithm
    r = SplitMix64(0)
    assert r.next() == 0xE220A8397B1DCDAF
    assert r.next() == 0x6E789E6AA1B965F4
    # reseed purity (test_engine.cpp:74-80) and divergence (:82-88)
    a, b = stream_rng(42, 9), stream_rng(42, 9)
    assert [a.next() for _ in range(1000)] == [b.next() for _ in range(1000)]
    a, b = stream_rng(42, 4), stream_rng(42, 5)
    assert any(a.next() != b.next() for _ in range(4))
    assert len({reseed(7, i) for i in range(10000)}) == 10000  # :90-94


def test_next_below_matches_oracle_and_edge_cases():
    L = oracle.lib()
    import ctypes as C
    rng = SplitMix64(123)
    st = C.c_uint64(123)
    bounds = [1, 2, 3, 7, 10, 1000, 2**32 - 1, 2**32 + 1, 2**63, 2**64 - 1, 2**64 - 3, (1 << 63) + 12345, 0]
    for k in range(3000):
        b = bounds[k % len(bounds)] if k < 600 else (mix64(k) >> (k % 64))
        assert rng.next_below(b) == L.or_next_below(C.byref(st), b)
    assert SplitMix64(5).next_below(0) == 0  # bound 0 returns 0 with one draw (rng.hpp:33-44)


# ----------------------------------------------------------------------------- kadabra.hpp scalars
def test_compute_omega_known_answers():
    # test_kadabra.cpp:112-130
    assert oracle.compute_omega(3, 0.1, 0.1) == 216
    assert oracle.compute_omega(3, 0.05, 0.1) == 861
    assert oracle.compute_omega(0, 0.1, 0.1) == oracle.compute_omega(3, 0.1, 0.1)
    assert oracle.compute_omega(1, 0.1, 0.1) == oracle.compute_omega(3, 0.1, 0.1)
    for bad in [(3, 1.0, 0.1), (3, 0.0, 0.1), (3, 0.1, 0.0)]:
        with pytest.raises(oracle.OracleError):
            oracle.compute_omega(*bad)


def test_fg_frozen_values():
    # test_util.hpp:266-267 (40-digit reference), test_kadabra.cpp:133-143
    kF, kG = 0.014795359120809299, 0.017213930684453299
    assert oracle.f_bound(0.1, 0.01, 1000, 2000) == pytest.approx(kF, rel=1e-12)
    assert oracle.g_bound(0.1, 0.01, 1000, 2000) == pytest.approx(kG, rel=1e-12)
    assert oracle.f_bound(0.0, 0.5, 1000, 3000) == 0.0
    assert oracle.f_bound(0.0, 0.01, 2000, 4000) == 0.0
    for args in [(0.1, 0.01, 10, 0), (-0.1, 0.01, 10, 10), (1.1, 0.01, 10, 10)]:
        with pytest.raises(oracle.OracleError):
            oracle.f_bound(*args)


def _ref_width(b, delta_v, omega, tau, upper):
    getcontext().prec = 50
    L = (Decimal(1) / Decimal(delta_v)).ln()
    t = Decimal(1) / 3 + (Decimal(omega) / tau if upper else -Decimal(omega) / tau)
    return (L / tau) * (t + (t * t + 2 * Decimal(b) * omega / L).sqrt())


def test_kadabra_check_vs_high_precision():
    # test_kadabra.cpp:197-216: agreement with an independent re-evaluation
    rng = SplitMix64(1234)
    true_count = 0
    for _ in range(300):
        n = 1 + rng.next_below(12)
        num = 1 + rng.next_below(50000)
        data = [rng.next_below(num + 1) for _ in range(n)]
        eps = 0.001 + rng.next_below(200) / 1000.0
        omega = 1 + rng.next_below(80000)
        delta_v = 0.0001 + rng.next_below(4000) / 10000.0
        got = oracle.kadabra_check(data, num, omega, eps, delta_v)
        want = num >= omega or all(
            _ref_width(Decimal(d) / num, delta_v, omega, num, False) <= Decimal(eps) and
            _ref_width(Decimal(d) / num, delta_v, omega, num, True) <= Decimal(eps) for d in data)
        assert got == want
        true_count += got
    assert 0 < true_count < 300


def test_max_count_equivalence():
    """The GPU evaluates the rule only at max_v data[v] (engine.cu). With uniform
    deltas this equals the per-vertex loop of kadabra_converged because f and g
    are monotone in b under IEEE round-to-nearest. Checked on 20k random states,
    including near-threshold ones."""
    rng = SplitMix64(99)
    agree = flips = 0
    for i in range(20000):
        n = 1 + rng.next_below(40)
        num = 1 + rng.next_below(200000)
        omega = num + 1 + rng.next_below(400000)
        hi = 1 + rng.next_below(num)
        data = [rng.next_below(hi + 1) for _ in range(n)]
        eps = [0.001, 0.005, 0.01, 0.05][i % 4] * (0.5 + rng.next_below(1000) / 1000.0)
        delta_v = 0.1 / (2.0 * n)
        full = oracle.kadabra_check(data, num, omega, eps, delta_v)
        at_max = oracle.kadabra_check([max(data)], num, omega, eps, delta_v)
        assert full == at_max
        flips += full
    assert flips > 100


# ----------------------------------------------------------------------------- graph.hpp
PARSE_CASES = [
    ("0 1\n1 2", 3, 2, [0, 1, 2]),                      # test_graph.cpp:12-17
    ("% c\n5 5\n5 7", 2, 1, [5, 7]),                    # :19-24
    ("0 1\n1 0\n0 1", 2, 1, [0, 1]),                    # :26-30
    ("# header\n0\t1\n1\t2\n", 3, 2, [0, 1, 2]),        # :32-36
    ("9 4\n4 2\n", 3, 2, [9, 4, 2]),                    # :38-41
    ("  \t\r\n7 8\r\n\n% x\n  # y\n8 7\n", 2, 1, [7, 8]),
    ("+3 4\n4 +5\n", 3, 2, [3, 4, 5]),
    ("-18446744073709551615 2\n", 2, 1, [1, 2]),        # istream >> uint64 negates mod 2^64
    ("4294967295 0\n", 2, 1, [4294967295, 0]),
    ("1 2", 2, 1, [1, 2]),
    ("3 3\n1 2\n", 3, 1, [3, 1, 2]),                    # self-loop line interns (isolated vertex)
]

PARSE_ERRORS = [
    ("0 1\nx y\n", "line 2: expected two vertex ids"),    # test_graph.cpp:43-50
    ("% nothing\n", "no vertices found in edge list"),    # :52-54
    ("", "no vertices found in edge list"),
    ("1\n", "line 1: expected two vertex ids"),
    ("1 2 3\n", "line 1: trailing token '3'"),
    ("1 2abc\n", "line 1: trailing token 'abc'"),
    ("12abc 5\n", "line 1: expected two vertex ids"),
    ("4294967296 1\n", "line 1: vertex id exceeds 2^32-1"),
    ("-1 2\n", "line 1: vertex id exceeds 2^32-1"),
    ("99999999999999999999 1\n", "line 1: expected two vertex ids"),
    ("0 1\n\x0b\n", "line 2: expected two vertex ids"),  # \v is not a blank-line char
    ("1.5 2\n", "line 1: expected two vertex ids"),
]


@pytest.mark.parametrize("text,n,m,ids", PARSE_CASES)
def test_parse_examples(text, n, m, ids):
    g = oracle.parse_text(text)
    assert g.n == n and g.nbrs.shape[0] == 2 * m
    assert list(g.original_ids) == ids


@pytest.mark.parametrize("text,msg", PARSE_ERRORS)
def test_parse_errors(text, msg):
    with pytest.raises(oracle.OracleError) as e:
        oracle.parse_text(text)
    assert str(e.value) == msg and e.value.code == 3


@pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference not present")
@pytest.mark.parametrize("text,msg", PARSE_ERRORS)
def test_parse_errors_match_reference(tmp_path, text, msg):
    import subprocess
    p = tmp_path / "g.edges"
    p.write_bytes(text.encode())
    r = subprocess.run([str(oracle.REF_DRIVER), "dub", "--graph", str(p)], capture_output=True, text=True)
    assert r.returncode == 1 and r.stderr.strip() == f"error: {msg}"


@pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference not present")
@pytest.mark.parametrize("text,n,m,ids", PARSE_CASES)
def test_parse_examples_match_reference(tmp_path, text, n, m, ids):
    p = tmp_path / "g.edges"
    p.write_bytes(text.encode())
    d = oracle.ref_dub(p)
    assert (d["n"], d["m"]) == (n, m)


def test_graph_invariants_and_components():
    from conftest import random_pairs
    rng = SplitMix64(2024)
    for it in range(300):  # test_graph.cpp:110-120 (union-find agreement)
        n = 2 + rng.next_below(63)
        pairs = random_pairs(n, 0.05, rng.next())
        if pairs.shape[0] == 0:
            continue
        g = oracle.from_pairs(pairs)
        off, nb = g.offsets, g.nbrs
        assert off[0] == 0 and off[-1] == nb.shape[0]
        for u in range(g.n):
            row = nb[off[u]:off[u + 1]]
            assert np.all(np.diff(row.astype(np.int64)) > 0) and u not in row
        lab, comps = oracle.components(g)
        parent = list(range(g.n))

        def find(x):
            while parent[x] != x:
                parent[x] = parent[parent[x]]
                x = parent[x]
            return x
        for u in range(g.n):
            for v in nb[off[u]:off[u + 1]]:
                parent[find(u)] = find(int(v))
        roots = [find(u) for u in range(g.n)]
        assert comps == len(set(roots))
        fwd = {}
        for a, b in zip(lab, roots):
            assert fwd.setdefault(a, b) == b


def test_dub_examples():
    # test_graph.cpp:123-154 (graphs built from dense edges)
    assert oracle.diameter_upper_bound(oracle.from_edges(5, [(0, i) for i in range(1, 5)])) == 2
    assert oracle.diameter_upper_bound(oracle.from_edges(4, [(i, j) for i in range(4) for j in range(i + 1, 4)])) == 2
    p5 = oracle.from_edges(5, [(i, i + 1) for i in range(4)])
    assert oracle.eccentricity(p5, 2) == 2 and oracle.diameter_upper_bound(p5) == 6
    assert oracle.diameter_upper_bound(oracle.from_edges(3, [(0, 1)])) == 2


# ----------------------------------------------------------------------------- goldens
def _graphs():
    import importlib.util
    spec = importlib.util.spec_from_file_location("make_golden", GOLD / "make_golden.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.graphs()


@pytest.fixture(scope="module")
def gold_graphs(tmp_path_factory):
    import hashlib
    d = tmp_path_factory.mktemp("gold")
    meta, _ = golden()
    out = {}
    for name, pairs in _graphs().items():
        path = d / f"{name}.edges"
        datasets.write_edge_list(path, pairs)
        assert hashlib.sha256(path.read_bytes()).hexdigest() == meta["graphs"][name]["sha256"], \
            f"generator drift for {name}"
        out[name] = (pairs, path)
    return out


def test_golden_dub(gold_graphs):
    meta, _ = golden()
    for name, (pairs, _) in gold_graphs.items():
        g = oracle.from_pairs(pairs)
        _, comps = oracle.components(g)
        want = meta["dub"][name]
        assert (g.n, g.nbrs.shape[0] // 2, comps, oracle.diameter_upper_bound(g)) == \
               (want["n"], want["m"], want["components"], want["diameter_bound"])


def test_golden_runs(gold_graphs):
    meta, arrays = golden()
    for run in meta["runs"]:
        g = oracle.from_pairs(gold_graphs[run["graph"]][0])
        r = oracle.estimate_bc(g, run["eps"], run["delta"], spf=run["spf"], seed=run["seed"],
                               nominal_threads=run["threads"])
        assert (r.tau, r.check_cycles, r.stop_epoch, r.omega, r.diameter_bound, r.reason) == \
               (run["tau"], run["check_cycles"], run["stop_epoch"], run["omega"], run["diameter_bound"],
                run["reason"]), run["key"]
        np.testing.assert_array_equal(r.counts, arrays["counts:" + run["key"]])
        assert oracle.fnv1a(r.counts) == run["counts_fnv1a"]


def test_golden_runs_threaded_oracle(gold_graphs):
    """or_estimate_bc_threads (frames sampled in parallel, folded in position
    order: how tests/golden/make_fullsize.py computes the full-size goldens the
    reference cannot produce) reproduces every reference golden run."""
    meta, arrays = golden()
    for run in meta["runs"]:
        g = oracle.from_pairs(gold_graphs[run["graph"]][0])
        r = oracle.estimate_bc(g, run["eps"], run["delta"], spf=run["spf"], seed=run["seed"],
                               nominal_threads=run["threads"], threads=3)
        assert (r.tau, r.check_cycles, r.stop_epoch, r.reason) == \
               (run["tau"], run["check_cycles"], run["stop_epoch"], run["reason"]), run["key"]
        np.testing.assert_array_equal(r.counts, arrays["counts:" + run["key"]])


def test_golden_frames_threaded_oracle(gold_graphs):
    meta, arrays = golden()
    for fr in meta["frames"]:
        g = oracle.from_pairs(gold_graphs[fr["graph"]][0])
        got = oracle.sample_frames(g, fr["seed"], fr["spf"], fr["first"], fr["count"], threads=3)
        assert [len(x) for x in got] == list(arrays["frames_len:" + fr["key"]])
        np.testing.assert_array_equal(np.concatenate(got), arrays["frames_ids:" + fr["key"]])


def test_golden_frames(gold_graphs):
    meta, arrays = golden()
    for fr in meta["frames"]:
        g = oracle.from_pairs(gold_graphs[fr["graph"]][0])
        got = oracle.sample_frames(g, fr["seed"], fr["spf"], fr["first"], fr["count"])
        lens = arrays["frames_len:" + fr["key"]]
        ids = arrays["frames_ids:" + fr["key"]]
        assert [len(x) for x in got] == list(lens)
        np.testing.assert_array_equal(np.concatenate(got) if got else ids, ids)


@pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference not present")
def test_live_reference_random_graphs(tmp_path):
    rng = SplitMix64(777)
    for it in range(6):
        n = 30 + rng.next_below(200)
        pairs = datasets.gen_gnm(n, n * (1 + rng.next_below(4)), rng.next(), lcc=bool(it % 2))
        path = tmp_path / f"g{it}.edges"
        datasets.write_edge_list(path, pairs)
        seed, spf = rng.next_below(1000), 1 + rng.next_below(4)
        want = oracle.ref_run(path, eps=0.05, delta=0.1, seed=seed, spf=spf, threads=3)
        g = oracle.parse_file(path)
        r = oracle.estimate_bc(g, 0.05, 0.1, spf=spf, seed=seed, nominal_threads=3)
        assert (r.tau, r.check_cycles, r.stop_epoch, oracle.fnv1a(r.counts)) == \
               (want["tau"], want["check_cycles"], want["stop_epoch"], want["counts_fnv1a"])
        frames = oracle.ref_frames(path, seed=seed, spf=spf, first=0, count=100, out_path=tmp_path / "f.bin")
        got = oracle.sample_frames(g, seed, spf, 0, 100)
        for a, b in zip(got, frames):
            np.testing.assert_array_equal(a, b)


def test_brandes_matches_apsp_definition():
    # exact normalized BC by brute force (test_util.hpp:186-205) on small graphs
    for name in ["path5", "star4", "cube", "diamond", "k23", "two_components", "er24"]:
        g = oracle.from_pairs(SMALL_GRAPHS[name]())
        n = g.n
        off, nb = g.offsets, g.nbrs
        dist = np.full((n, n), -1)
        sig = np.zeros((n, n))
        for s in range(n):
            dist[s, s] = 0
            sig[s, s] = 1
            q = [s]
            for u in q:
                for v in nb[off[u]:off[u + 1]]:
                    if dist[s, v] < 0:
                        dist[s, v] = dist[s, u] + 1
                        q.append(int(v))
                    if dist[s, v] == dist[s, u] + 1:
                        sig[s, v] += sig[s, u]
        bc = np.zeros(n)
        for s in range(n):
            for t in range(n):
                if s == t or dist[s, t] < 0:
                    continue
                for v in range(n):
                    if v not in (s, t) and dist[s, v] >= 0 and dist[v, t] >= 0 and dist[s, v] + dist[v, t] == dist[s, t]:
                        bc[v] += sig[s, v] * sig[v, t] / sig[s, t]
        bc /= n * (n - 1)
        np.testing.assert_allclose(oracle.brandes(g, 2), bc, rtol=1e-12, atol=1e-15)


def test_epoch_mode_is_indexed_prefix():
    """The epoch restatement at tau = k*B holds exactly the increments of the
    first tau one-sample frames of the indexed keying (stream_rng(seed, i))."""
    g = oracle.from_pairs(SMALL_GRAPHS["er100"]())
    e = oracle.estimate_bc(g, 0.05, 0.1, mode=oracle.MODE_EPOCH, epoch_samples=100, seed=3)
    assert e.tau % 100 == 0 and e.check_cycles == e.tau // 100
    want = np.zeros(g.n, np.uint64)
    for inc in oracle.sample_frames(g, 3, 1, 0, e.tau):
        np.add.at(want, inc, 1)
    np.testing.assert_array_equal(e.counts, want)


@pytest.mark.parametrize("name", ["c1_er", "c2_rmat18", "c3_ba", "c4_grid"])
def test_generators_match_product(name):
    """oracle/gen.c (what bench.py's reference arm generates its graph with, so
    that arm never loads libadsb.so) emits the product generators' exact edge
    sequence, LCC included."""
    w = datasets.CONFIGS[name]
    np.testing.assert_array_equal(oracle.gen_pairs(w.kind, w.params), datasets.pairs(name))


def test_generators_match_product_small():
    cases = [("gnm", (300, 900, 5), datasets.gen_gnm), ("rmat", (10, 8, 0.57, 0.19, 0.19, 3), datasets.gen_rmat),
             ("ba", (500, 3, 9), datasets.gen_ba), ("grid", (40, 30, 0.3, 2), datasets.gen_grid)]
    for kind, params, fn in cases:
        np.testing.assert_array_equal(oracle.gen_pairs(kind, params), fn(*params))
    for kind, params, fn in cases:
        if kind != "ba":
            np.testing.assert_array_equal(oracle.gen_pairs(kind, params, lcc=False), fn(*params, lcc=False))


def test_dense_edges_file_roundtrip(tmp_path):
    """The --graph-bin input of ref_driver: first-appearance dense ids, i.e. the
    ids parse_edge_list assigns (graph.hpp:98-123)."""
    pairs = datasets.gen_rmat(9, 8, 0.57, 0.19, 0.19, 4)
    path = tmp_path / "g.bin"
    oracle.write_dense_edges(path, pairs)
    raw = path.read_bytes()
    n = int(np.frombuffer(raw, "<u4", 1, 0)[0])
    m = int(np.frombuffer(raw, "<u8", 1, 4)[0])
    dense = np.frombuffer(raw, "<u4", 2 * m, 12)
    g = oracle.from_pairs(pairs)
    assert n == g.n and m == pairs.shape[0] // 2
    ids = g.original_ids
    np.testing.assert_array_equal(ids[dense], pairs)

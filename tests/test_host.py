"""CPU tests of the product's host side and its C ABI (no GPU needed).

The host ingestion (parse_edge_list / from_edges / CSR) and the scalar rules
run on the CPU by design; they are compared with the oracle here. Everything
that traverses the graph is GPU-only and covered by test_gpu_parity.py.
"""
from __future__ import annotations

import ctypes as C
import json
import re
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_1903_09422_b200 import CudaError, InvalidArgument, ParseError, _lib, adsamp, datasets, kadabra

from conftest import SMALL_GRAPHS
from test_oracle import PARSE_CASES, PARSE_ERRORS

ROOT = Path(__file__).resolve().parents[1]


def test_c_abi_exports_every_declared_symbol():
    header = (ROOT / "include" / "adsb.h").read_text()
    declared = set(re.findall(r"\b(adsb_[a-z_0-9]+)\s*\(", header))
    lib = C.CDLL(str(_lib.LIB_PATH))
    missing = [name for name in sorted(declared) if not hasattr(lib, name)]
    assert not missing, missing
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    assert _lib.lib().adsb_abi_version() == 2


def test_struct_layouts():
    """ctypes mirrors of adsb.h's structs match the C compiler's layout."""
    assert C.sizeof(_lib.Config) == 96
    assert C.sizeof(_lib.Stats) == 168
    assert C.sizeof(_lib.HostCollectives) == 24


@pytest.mark.parametrize("text,n,m,ids", PARSE_CASES)
def test_parse_examples(text, n, m, ids):
    p = adsamp.parse_edge_list(text)
    o = oracle.parse_text(text)
    assert p.graph.num_vertices() == n and p.graph.num_edges() == m
    assert list(p.original_ids) == ids
    np.testing.assert_array_equal(p.graph.offsets(), o.offsets)
    np.testing.assert_array_equal(p.graph.neighbor_list(), o.nbrs)


@pytest.mark.parametrize("text,msg", PARSE_ERRORS)
def test_parse_errors(text, msg):
    with pytest.raises(ParseError) as e:
        adsamp.parse_edge_list(text)
    assert str(e.value) == msg


def _big_edge_list(lines: int, seed: int = 5) -> list[str]:
    rng = np.random.default_rng(seed)
    a = rng.integers(0, 40000, size=lines) * 7 + 3  # sparse ids: exercises the first-appearance remap
    b = rng.integers(0, 40000, size=lines) * 7 + 3
    out = [f"{x} {y}" for x, y in zip(a.tolist(), b.tolist())]
    for i in range(0, lines, 997):
        out[i] = "# comment " + out[i]  # comments and blank lines keep their line numbers
    for i in range(5, lines, 1999):
        out[i] = ""
    return out


def test_parse_parallel_chunks_match_oracle():
    """Texts over 4 MB are parsed in line-aligned chunks on every host thread;
    the CSR, the id remap and the error line numbers equal a sequential parse."""
    lines = _big_edge_list(400_000)
    text = "\n".join(lines) + "\n"
    assert len(text) > (4 << 20)
    p = adsamp.parse_edge_list(text)
    o = oracle.parse_text(text)
    np.testing.assert_array_equal(p.graph.offsets(), o.offsets)
    np.testing.assert_array_equal(p.graph.neighbor_list(), o.nbrs)
    np.testing.assert_array_equal(p.original_ids, o.original_ids)
    for bad_line, bad in [(350_001, "12 x"), (123_457, "1 2 3"), (399_990, "5 99999999999")]:
        broken = list(lines)
        broken[bad_line - 1] = bad
        later = bad_line + 20  # a second, later error must not win
        if later <= len(broken):
            broken[later - 1] = "only_one"
        with pytest.raises(ParseError) as e:
            adsamp.parse_edge_list("\n".join(broken))
        with pytest.raises(Exception) as eo:
            oracle.parse_text("\n".join(broken))
        assert str(e.value).startswith(f"line {bad_line}: "), str(e.value)
        assert str(e.value) == str(eo.value)


def test_parse_file_and_pairs_agree(tmp_path):
    for name in ["er100", "cube", "two_components"]:
        pairs = SMALL_GRAPHS[name]().reshape(-1)
        path = tmp_path / f"{name}.edges"
        datasets.write_edge_list(path, pairs)
        a = adsamp.parse_edge_list_file(path)
        b = adsamp.graph_from_pairs(pairs)
        o = oracle.parse_file(path)
        for g in (a, b):
            np.testing.assert_array_equal(g.graph.offsets(), o.offsets)
            np.testing.assert_array_equal(g.graph.neighbor_list(), o.nbrs)
            np.testing.assert_array_equal(g.original_ids, o.original_ids)


def test_c1_ingestion_matches_oracle():
    pairs = datasets.pairs("c1_er")
    g = adsamp.graph_from_pairs(pairs)
    o = oracle.from_pairs(pairs)
    assert g.graph.num_vertices() == 10_000 and g.graph.num_edges() == 50_000
    np.testing.assert_array_equal(g.graph.offsets(), o.offsets)
    np.testing.assert_array_equal(g.graph.neighbor_list(), o.nbrs)
    np.testing.assert_array_equal(g.original_ids, o.original_ids)


def test_from_edges_and_csr_validation():
    g = adsamp.Graph.from_edges(4, [(0, 1), (1, 0), (2, 2), (3, 1)])
    assert g.num_vertices() == 4 and g.num_edges() == 2
    assert list(g.neighbors(1)) == [0, 3]
    with pytest.raises(InvalidArgument):
        adsamp.Graph.from_edges(2, [(0, 5)])
    h = adsamp.Graph.from_csr(4, g.offsets(), g.neighbor_list())
    np.testing.assert_array_equal(h.neighbor_list(), g.neighbor_list())
    with pytest.raises(InvalidArgument):
        adsamp.Graph.from_csr(2, [0, 1, 2], [1, 1])  # self loop at 1
    with pytest.raises(InvalidArgument):
        adsamp.Graph.from_csr(3, [0, 2, 2, 2], [2, 1])  # not ascending


def test_large_csr_validation_on_host_workers():
    """from_csr above the parallel threshold runs on the persistent host
    workers: a valid CSR round-trips, and a defect in any range (one per
    worker range tried) is reported, repeatedly (the pool is reused)."""
    pairs = datasets.gen_gnm(60000, 300000, 3)
    g = adsamp.graph_from_pairs(pairs).graph
    off, nb = g.offsets().copy(), g.neighbor_list().copy()
    assert nb.size >= 262144
    for _ in range(3):
        h = adsamp.Graph.from_csr(g.num_vertices(), off, nb)
        np.testing.assert_array_equal(h.offsets(), off)
        np.testing.assert_array_equal(h.neighbor_list(), nb)
    n = g.num_vertices()
    for frac in (0.02, 0.5, 0.97):
        u = int(np.searchsorted(off, int(frac * nb.size), side="right")) - 1
        while off[u + 1] - off[u] < 2:
            u += 1
        bad = nb.copy()
        bad[off[u] + 1] = bad[off[u]]  # duplicate neighbour
        with pytest.raises(InvalidArgument):
            adsamp.Graph.from_csr(n, off, bad)
        bad = nb.copy()
        bad[off[u]] = u  # self loop
        with pytest.raises(InvalidArgument):
            adsamp.Graph.from_csr(n, off, bad)


def test_serialize_and_renumbering():
    # graph.hpp:140-144 writes dense ids; re-parsing renumbers them by first
    # appearance, so the round trip is NOT the identity in general (the
    # reference's own test_graph.cpp:76-89 asserts it and would fail).
    g = adsamp.Graph.from_edges(3, [(0, 2), (1, 2)])
    text = adsamp.serialize_edge_list(g)
    assert text == "0 2\n1 2\n"
    back = adsamp.parse_edge_list(text)
    assert list(back.original_ids) == [0, 2, 1]
    assert list(back.graph.neighbor_list()) != list(g.neighbor_list())


def test_generators_are_deterministic_and_sized():
    a, b = datasets.gen_rmat(10, 8, 0.57, 0.19, 0.19, 5), datasets.gen_rmat(10, 8, 0.57, 0.19, 0.19, 5)
    np.testing.assert_array_equal(a, b)
    ba = datasets.gen_ba(500, 3, 2)
    assert ba.shape[0] == 2 * (3 * 4 // 2 + (500 - 4) * 3)
    grid = datasets.gen_grid(16, 16, 0.0, 0)
    assert grid.shape[0] == 2 * 480
    c1 = datasets.pairs("c1_er")
    assert c1.shape[0] == 100_000


def test_scalar_rules_match_oracle():
    for dub in [0, 1, 3, 8, 12, 8182, 10**6]:
        for eps in [0.001, 0.005, 0.01, 0.1]:
            assert kadabra.compute_omega(dub, eps, 0.1) == oracle.compute_omega(dub, eps, 0.1)
    rng = adsamp.SplitMix64(5)
    for _ in range(500):
        b = rng.next_below(10**6) / 10**6
        dv = (1 + rng.next_below(10**6)) / 10**7
        om, tau = 1 + rng.next_below(10**5), 1 + rng.next_below(10**5)
        assert kadabra.f_bound(b, dv, om, tau) == oracle.f_bound(b, dv, om, tau)
        assert kadabra.g_bound(b, dv, om, tau) == oracle.g_bound(b, dv, om, tau)
    with pytest.raises(ValueError):
        kadabra.f_bound(0.1, 0.01, 10, 0)
    with pytest.raises(ValueError):
        kadabra.compute_omega(3, 1.0, 0.1)
    d = np.array([400, 100, 0], np.uint64)
    assert kadabra.kadabra_check(d, 500, 500, 0.0001, 0.1)  # omega cap (test_kadabra.cpp:178-182)


def test_engine_helpers():
    # test_engine.cpp:50-60, :62-72, :220-229
    xi32 = np.log(100.0) / np.log(32.0)
    assert adsamp.check_budget(1000, 32, xi32) == 10
    assert adsamp.check_budget(1000, 1, 1.3285) == 1000
    assert adsamp.check_budget(1000, 4, 1.3285) == 159
    assert adsamp.check_budget(1, 64, 2.0) == 1
    with pytest.raises(InvalidArgument):
        adsamp.check_budget(0, 1, 1.0)
    assert adsamp.shared_frame_target(5, 2) == 1
    assert adsamp.indexed_frame_index(2, 1, 4) == 9
    c = adsamp.ReservationCounter()
    assert [adsamp.reserve_indices(c, 4, 2) for _ in range(5)] == \
           [[0, 4, 8], [1, 5, 9], [2, 6, 10], [3, 7, 11], [12, 16, 20]]
    cfg = adsamp.EngineConfig(threads=2, variant=adsamp.Variant.shared, frame_groups=3)
    with pytest.raises(InvalidArgument):
        cfg.validate()
    assert adsamp.parse_variant("indexed") == adsamp.Variant.indexed
    with pytest.raises(InvalidArgument):
        adsamp.parse_variant("bogus")


def _cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_cuda_available(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback_without_gpu():
    g = adsamp.Graph.from_edges(3, [(0, 1), (1, 2)])
    with pytest.raises(CudaError, match="no CUDA device"):
        kadabra.estimate_bc(g, 0.1, 0.1, adsamp.EngineConfig(variant=adsamp.Variant.indexed))
    with pytest.raises(CudaError):
        adsamp.connected_components(g)


def test_bench_reference_arm_loads_no_product_code():
    """bench.py --impl reference times the compiled reference on a graph made by
    oracle/gen.c: the process must not map libadsb.so, and its metric string
    must equal the GPU arm's (the driver compares them verbatim)."""
    import subprocess
    import sys
    code = (
        "import sys, runpy, json, io, contextlib\n"
        "sys.argv=['bench.py','--impl','reference','--config','c1_er','--steps','1','--warmup','3']\n"
        "buf=io.StringIO()\n"
        "with contextlib.redirect_stdout(buf):\n"
        "    runpy.run_path('bench.py', run_name='__main__')\n"
        "line=json.loads(buf.getvalue().strip().splitlines()[-1])\n"
        "print(json.dumps({'metric': line['metric'], 'kind': line['cpu_baseline']['kind'],\n"
        "  'libadsb': 'libadsb' in open('/proc/self/maps').read()}))\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=str(ROOT), capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    got = json.loads(out.stdout.strip().splitlines()[-1])
    assert got["libadsb"] is False
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_1903_09422_b200 import datasets
    assert got["metric"] == bench.metric_name(datasets.CONFIGS["c1_er"])


def test_cpp_dropin_header_source_compatible(tmp_path):
    """A reference caller's code compiles unchanged against adsamp_b200.hpp:
    estimate_bc takes an AuditSink* (kadabra.hpp:308-309), EngineConfig has
    validate() (engine.hpp:97-105), RunResult has queue (engine.hpp:163-171)."""
    import subprocess
    src = tmp_path / "caller.cpp"
    src.write_text(r'''
#include "adsamp_b200.hpp"
using namespace adsamp_b200;
int main() {
    EngineConfig cfg;
    cfg.variant = Variant::indexed;
    cfg.bounded_memory = true;
    cfg.validate();
    bool threw = false;
    try { EngineConfig bad; bad.threads = 0; bad.validate(); } catch (const std::invalid_argument&) { threw = true; }
    if (!threw) return 1;
    AuditSink* sink = nullptr;
    auto parsed = parse_edge_list(std::string("0 1\n1 2\n"));
    if (false) {
        kadabra::BcResult r = kadabra::estimate_bc(parsed.graph, 0.1, 0.1, cfg, sink);
        return static_cast<int>(r.run.queue.max_depth + r.run.queue.high_water_exceeded);
    }
    return parsed.graph.num_vertices() == 3 ? 0 : 2;
}
''')
    exe = tmp_path / "caller"
    pkg = ROOT / "paper_1903_09422_b200"
    out = subprocess.run(["g++", "-std=c++20", f"-I{ROOT / 'include'}", str(src), "-o", str(exe), f"-L{pkg}",
                          "-ladsb", f"-Wl,-rpath,{pkg}"], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True)
    assert run.returncode == 0, (run.returncode, run.stderr)


REF_DATA = Path("/root/reference/proj/data")


@pytest.mark.skipif(not REF_DATA.exists(), reason="reference data fixtures not present")
@pytest.mark.parametrize("name", ["toy_path.edges", "grid16.edges"])
def test_reference_data_fixtures_ingest(name):
    """The reference's own fixture files (proj/data/) through the product's
    parser, the oracle and the compiled reference: same ids, same CSR, same D_ub."""
    path = REF_DATA / name
    p = adsamp.parse_edge_list_file(path)
    o = oracle.parse_file(path)
    np.testing.assert_array_equal(p.graph.offsets(), o.offsets)
    np.testing.assert_array_equal(p.graph.neighbor_list(), o.nbrs)
    assert list(p.original_ids) == list(o.original_ids)
    if oracle.ref_available():
        d = oracle.ref_dub(path)
        assert (d["n"], d["m"]) == (p.graph.num_vertices(), p.graph.num_edges())
        assert d["diameter_bound"] == oracle.diameter_upper_bound(o)


def test_graph_cache_round_trip(tmp_path):
    """Binary CSR cache: the identical graph (CSR, dense ids,
    original ids) comes back; damage and truncation raise ParseError."""
    for text in ["5 9\n9 7\n7 5\n% c\n1000000 5\n", "0 1\n1 2\n2 0\n"]:
        p = adsamp.parse_edge_list(text)
        path = tmp_path / "g.adsbcsr"
        adsamp.save_graph(p, path)
        q = adsamp.load_graph(path)
        np.testing.assert_array_equal(q.graph.offsets(), p.graph.offsets())
        np.testing.assert_array_equal(q.graph.neighbor_list(), p.graph.neighbor_list())
        np.testing.assert_array_equal(q.original_ids, p.original_ids)
    big = adsamp.graph_from_pairs(datasets.gen_rmat(14, 16, 0.57, 0.19, 0.19, 2))
    path = tmp_path / "big.adsbcsr"
    adsamp.save_graph(big, path)
    q = adsamp.load_graph(path)
    np.testing.assert_array_equal(q.graph.neighbor_list(), big.graph.neighbor_list())
    np.testing.assert_array_equal(q.original_ids, big.original_ids)
    raw = bytearray(path.read_bytes())
    raw[len(raw) // 2] ^= 0x40
    bad = tmp_path / "bad.adsbcsr"
    bad.write_bytes(bytes(raw))
    with pytest.raises(ParseError, match="damaged"):
        adsamp.load_graph(bad)
    bad.write_bytes(bytes(raw[: len(raw) - 8]))
    with pytest.raises(ParseError, match="truncated"):
        adsamp.load_graph(bad)
    bad.write_bytes(b"not a cache at all, definitely not" * 4)
    with pytest.raises(ParseError, match="not an adsb graph cache"):
        adsamp.load_graph(bad)


def test_datasets_graph_cache(tmp_path):
    a = datasets.graph("c1_er", cache_dir=tmp_path)
    assert (tmp_path / "c1_er.adsbcsr").exists()
    b = datasets.graph("c1_er", cache_dir=tmp_path)
    np.testing.assert_array_equal(a.graph.neighbor_list(), b.graph.neighbor_list())
    np.testing.assert_array_equal(a.original_ids, b.original_ids)

"""The multi-rank engine itself (engine.cu), world size 2, on one GPU.

Two processes each run libadsb's real multi-GPU code — rank sharding of frame
positions and sample indices, the all-gather of per-sample increments with
padding, the ordered cutoff on every rank, the barrier variant's all-reduce
of the n-length count vector, and the rank-invariant batch sizing — over the
host-callback transport (adsb_comm_init_host, torch.distributed gloo), since
a gpurun box has a single GPU. No kernel waits on the other rank (only the
host does), so two ranks sharing the GPU is safe. Every rank's result must
equal the one-process run bit for bit (tau, check cycles, every count) and
the CPU oracle's.
"""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_1903_09422_b200 import adsamp, datasets
from paper_1903_09422_b200.adsamp import EngineConfig, Variant
from paper_1903_09422_b200.kadabra import estimate_bc

pytestmark = pytest.mark.gpu
HERE = Path(__file__).resolve().parent

# (name, generator, eps, variant, extra config)
CASES = [
    ("c1_indexed", "c1", 0.02, "indexed", {"samples_per_frame": 1}),
    ("c1_indexed_spf7", "c1", 0.02, "indexed", {"samples_per_frame": 7}),
    ("c1_indexed_bounded", "c1", 0.02, "indexed", {"samples_per_frame": 1, "bounded_memory": True,
                                                   "reservation_block": 2}),
    ("c1_shared", "c1", 0.02, "shared", {"epoch_samples": 512}),
    ("c1_barrier", "c1", 0.02, "barrier", {"check_interval": 1000}),
    ("rmat14_shared", "rmat14", 0.02, "shared", {}),
    ("rmat14_indexed", "rmat14", 0.02, "indexed", {"samples_per_frame": 1}),
    ("rmat14_barrier", "rmat14", 0.02, "barrier", {"epoch_samples": 2048}),
    ("grid96_indexed", "grid96", 0.05, "indexed", {"samples_per_frame": 1}),
    ("grid96_shared", "grid96", 0.05, "shared", {"epoch_samples": 256}),
]


def graph_pairs(kind: str) -> np.ndarray:
    if kind == "c1":
        return datasets.pairs("c1_er")
    if kind == "rmat14":
        return datasets.gen_rmat(14, 16, 0.57, 0.19, 0.19, 3)
    if kind == "grid96":
        return datasets.gen_grid(96, 96, 0.1, 5)
    raise KeyError(kind)


def config(variant: str, extra: dict, comm=None) -> EngineConfig:
    return EngineConfig(variant=Variant[variant], threads=8, base_seed=42, device=0, comm=comm, **extra)


def summary(r) -> dict:
    return {"tau": int(r.tau), "cycles": int(r.run.check_cycles), "stop_epoch": int(r.run.stop_epoch),
            "reason": r.reason.name, "fnv": oracle.fnv1a(r.run.data), "omega": int(r.omega)}


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def world2(tmp_path_factory):
    """Run every case on 2 ranks (two processes, host transport); {case: [rank0, rank1]}."""
    out_dir = tmp_path_factory.mktemp("mr")
    port = _free_port()
    procs = []
    for rank in range(2):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(HERE / "_multirank_worker.py"), str(out_dir)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = [p.communicate(timeout=900)[0] for p in procs]
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log[-4000:]
    res = [json.loads((out_dir / f"rank{r}.json").read_text()) for r in range(2)]
    return {k: [res[0][k], res[1][k]] for k in res[0]}


@pytest.mark.parametrize("name,kind,eps,variant,extra", CASES, ids=[c[0] for c in CASES])
def test_world2_equals_world1(world2, name, kind, eps, variant, extra):
    pg = adsamp.graph_from_pairs(graph_pairs(kind))
    single = summary(estimate_bc(pg.graph, eps, 0.1, config(variant, extra)))
    r0, r1 = world2[name]
    assert r0["world"] == 2 and r1["world"] == 2
    for r in (r0, r1):
        got = {k: r[k] for k in single}
        assert got == single, (name, r["rank"], got, single)


@pytest.mark.parametrize("name,kind,eps,variant,extra", [c for c in CASES if c[1] != "rmat14"],
                         ids=[c[0] for c in CASES if c[1] != "rmat14"])
def test_world2_equals_oracle(world2, name, kind, eps, variant, extra):
    og = oracle.from_pairs(graph_pairs(kind))
    if variant == "indexed":
        o = oracle.estimate_bc(og, eps, 0.1, spf=extra["samples_per_frame"], seed=42, nominal_threads=8, threads=4)
    else:
        B = extra.get("epoch_samples") or (extra.get("check_interval", 1000) if variant == "barrier" else 1024)
        o = oracle.estimate_bc(og, eps, 0.1, mode=oracle.MODE_EPOCH, epoch_samples=B, seed=42, threads=4)
    r0 = world2[name][0]
    assert (r0["tau"], r0["cycles"], r0["fnv"]) == (o.tau, o.check_cycles, oracle.fnv1a(o.counts)), name

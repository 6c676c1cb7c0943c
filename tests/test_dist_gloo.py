"""Multi-rank decomposition of both pipelines, world_size 2 over gloo (CPU).

engine.cu shards work across GPUs as `position = first + item * world + rank`
and combines it with one collective per epoch (all-reduce of the n-length
count vector) or per batch (all-gather of the (vertex, frame) events followed
by the ordered cutoff on every rank). Here each rank computes its shard with
the CPU oracle, the same collectives run over gloo, and the decisions must be
identical on both ranks and equal to the single-process result — i.e. the
decomposition is rank-count invariant, which is what makes the NCCL path
bit-exact across 1/2/4/8 GPUs.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1903_09422_b200 import kadabra

from conftest import SMALL_GRAPHS

EPS, DELTA, SEED = 0.05, 0.1, 17


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup():
    pairs = SMALL_GRAPHS["er100"]()
    g = oracle.from_pairs(pairs)
    omega = oracle.compute_omega(oracle.diameter_upper_bound(g), EPS, DELTA)
    return g, omega


def _rule(counts: np.ndarray, tau: int, omega: int) -> bool:
    """The product's host kadabra_check (kadabra.hpp:148-151, uniform deltas)."""
    return kadabra.kadabra_check(counts, tau, omega, EPS, DELTA)


def _epoch_rank(rank: int, world: int, port: int, B: int, out):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g, omega = _setup()
    total = np.zeros(g.n, np.int64)
    e = 0
    while True:
        local = np.zeros(g.n, np.int64)
        share = (B - rank + world - 1) // world
        for item in range(share):
            pos = e * B + item * world + rank
            for v in oracle.sample_frames(g, SEED, 1, pos, 1)[0]:
                local[v] += 1
        t = torch.from_numpy(local)
        dist.all_reduce(t)  # the NCCL all-reduce of engine.cu's epoch check
        total += t.numpy()
        tau = (e + 1) * B
        stop = _rule(total.astype(np.uint64), tau, omega)
        flags = [None] * world
        dist.all_gather_object(flags, stop)
        assert len(set(flags)) == 1
        if stop:
            break
        e += 1
    out[rank] = (tau, e + 1, total.tolist())
    dist.destroy_process_group()


def _cutoff(events: np.ndarray, base: np.ndarray, frames: int, done: int, omega: int) -> int | None:
    """engine.cu K4: sort (v, frame), running count per vertex, per-frame max,
    prefix max, first frame whose prefix passes the rule."""
    ev = np.sort(events[events != np.iinfo(np.uint64).max])
    v = (ev >> np.uint64(32)).astype(np.int64)
    f = (ev & np.uint64(0xFFFFFFFF)).astype(np.int64)
    first = np.searchsorted(v, v, side="left")
    value = base[v] + (np.arange(v.shape[0]) - first) + 1
    fmax = np.zeros(frames, np.int64)
    np.maximum.at(fmax, f, value)
    run = np.maximum.accumulate(np.maximum(fmax, base.max()))
    for k in range(frames):
        if _max_rule(int(run[k]), done + k + 1, omega, base.shape[0]):
            return k
    return None


def _max_rule(mx: int, tau: int, omega: int, n: int) -> bool:
    """kadabra_check on a state whose largest count is mx (deltas delta/(2n));
    equal to the per-vertex rule by monotonicity (test_oracle.py)."""
    arr = np.zeros(n, np.uint64)
    arr[0] = mx
    return _rule(arr, tau, omega)


def _det_rank(rank: int, world: int, port: int, F: int, out):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g, omega = _setup()
    total = np.zeros(g.n, np.int64)
    done = 0
    while True:
        ev = []
        for item in range((F - rank + world - 1) // world):
            f = item * world + rank
            for v in oracle.sample_frames(g, SEED, 1, done + f, 1)[0]:
                ev.append((int(v) << 32) | f)
        mine = torch.tensor([len(ev)], dtype=torch.int64)
        dist.all_reduce(mine, op=dist.ReduceOp.MAX)
        pad = np.full(int(mine.item()), np.iinfo(np.uint64).max, np.uint64)
        pad[: len(ev)] = np.array(ev, np.uint64)
        gathered = [torch.zeros(pad.shape[0], dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(pad.view(np.int64)))
        allev = np.concatenate([t.numpy().view(np.uint64) for t in gathered])
        k = _cutoff(allev, total, F, done, omega)
        limit = F - 1 if k is None else k
        real = allev[allev != np.iinfo(np.uint64).max]
        keep = (real & np.uint64(0xFFFFFFFF)).astype(np.int64) <= limit
        np.add.at(total, (real[keep] >> np.uint64(32)).astype(np.int64), 1)
        done += limit + 1
        if k is not None:
            break
    out[rank] = (done, total.tolist())
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [50, 128])
def test_epoch_decomposition_world2(B):
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_epoch_rank, args=(2, port, B, out), nprocs=2, join=True)
        r0, r1 = out[0], out[1]
    assert r0 == r1
    g, _ = _setup()
    single = oracle.estimate_bc(g, EPS, DELTA, mode=oracle.MODE_EPOCH, epoch_samples=B, seed=SEED)
    assert (r0[0], r0[1]) == (single.tau, single.check_cycles)
    np.testing.assert_array_equal(np.array(r0[2], np.uint64), single.counts)


def test_deterministic_decomposition_world2():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_det_rank, args=(2, port, 257, out), nprocs=2, join=True)
        r0, r1 = out[0], out[1]
    assert r0 == r1
    g, _ = _setup()
    single = oracle.estimate_bc(g, EPS, DELTA, spf=1, seed=SEED)
    assert r0[0] == single.tau == single.check_cycles
    np.testing.assert_array_equal(np.array(r0[1], np.uint64), single.counts)

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build libadsb.so (nvcc cross-compiles without a GPU) and the oracle once."""
    from paper_1903_09422_b200 import build as b
    if not b.LIB.exists():
        b.build()
    import oracle
    if not oracle.LIB_PATH.exists():
        oracle.build()
    yield


@pytest.fixture(scope="session")
def tmpdir_session(tmp_path_factory):
    return tmp_path_factory.mktemp("adsb")


# --------------------------------------------------------------------------- small graph fixtures
def path_pairs(k):
    return np.array([(i, i + 1) for i in range(k - 1)], dtype=np.uint64)


def cycle_pairs(k):
    return np.array([(i, (i + 1) % k) for i in range(k)], dtype=np.uint64)


def star_pairs(leaves):
    return np.array([(0, i) for i in range(1, leaves + 1)], dtype=np.uint64)


def complete_pairs(k):
    return np.array([(i, j) for i in range(k) for j in range(i + 1, k)], dtype=np.uint64)


def bipartite_pairs(a, b):
    return np.array([(i, a + j) for i in range(a) for j in range(b)], dtype=np.uint64)


def cube_pairs():
    return np.array([(u, u ^ (1 << bit)) for u in range(8) for bit in range(3) if u < u ^ (1 << bit)],
                    dtype=np.uint64)


def diamond_pairs():
    return np.array([(0, 1), (0, 2), (1, 2), (1, 3), (2, 3)], dtype=np.uint64)


def random_pairs(n, p, seed):
    """tests/test_util.hpp:84-92 G(n, p) edge order, restated."""
    from paper_1903_09422_b200.adsamp import SplitMix64
    rng = SplitMix64(seed)
    thr = int(p * 18446744073709551616.0)
    out = []
    for i in range(n):
        for j in range(i + 1, n):
            if rng.next() < thr:
                out.append((i, j))
    return np.array(out, dtype=np.uint64).reshape(-1, 2)


SMALL_GRAPHS = {
    "path3": lambda: path_pairs(3),
    "path5": lambda: path_pairs(5),
    "cycle4": lambda: cycle_pairs(4),
    "star4": lambda: star_pairs(4),
    "k5": lambda: complete_pairs(5),
    "k23": lambda: bipartite_pairs(2, 3),
    "cube": cube_pairs,
    "diamond": diamond_pairs,
    "two_components": lambda: np.array([(0, 1), (1, 2), (3, 4), (4, 5)], dtype=np.uint64),
    "er100": lambda: random_pairs(100, 0.05, 20240501),
    "er24": lambda: random_pairs(24, 0.15, 77),
}

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def c0_tree():
    import gen
    return gen.scene_c0()


@pytest.fixture(scope="session")
def c1_tree():
    import gen
    return gen.scene_c1()


def rng(seed):
    return np.random.Generator(np.random.Philox(key=seed))


def make_tree(child, sigma, sh, depth, sh_degree, bbox_min=(-1.0, -1.0, -1.0), edge=2.0):
    import gen
    return gen.Tree(depth, np.asarray(bbox_min, np.float32), float(edge), sh_degree,
                    np.asarray(child, np.uint32).reshape(-1, 8), np.asarray(sigma, np.float32),
                    np.asarray(sh, np.float32).reshape(len(sigma), (sh_degree + 1) ** 2, 3))


def full_depth1(sigma, sh_degree=0, k=0.0):
    """Depth-1 tree whose 8 octants are leaves 0..7 (octant order)."""
    child = [[(2 << 30) | o for o in range(8)]]
    B = (sh_degree + 1) ** 2
    sig = np.broadcast_to(np.asarray(sigma, np.float32), (8,))
    sh = np.broadcast_to(np.asarray(k, np.float32), (8, B, 3))
    return make_tree(child, sig, sh, 1, sh_degree)


def slab_chord(o, d, lo=-1.0, hi=1.0):
    """Textbook slab test (independent of the oracle): returns (t_near, t_far) or None."""
    o, d = np.asarray(o, float), np.asarray(d, float)
    d = d / np.linalg.norm(d)
    tn, tf = 0.0, np.inf
    for k in range(3):
        if d[k] == 0:
            if not (lo <= o[k] <= hi):
                return None
            continue
        a, b = (lo - o[k]) / d[k], (hi - o[k]) / d[k]
        tn, tf = max(tn, min(a, b)), min(tf, max(a, b))
    return (tn, tf) if tf > tn else None

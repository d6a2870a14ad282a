"""Pins for the oracle's ray-voxel segment extraction (§4.2).

* recursive ordered descent == brute force over all leaves (random mixed-depth trees)
* uniform / sparse single-depth trees == dense-grid Amanatides-Woo DDA written here
* segment midpoints locate (by an independent child-table walk) the segment's leaf
* sum of deltas over a full uniform tree == the analytic slab chord
"""
import numpy as np
import pytest

import gen
from conftest import rng, slab_chord


def _rays(seed, n, inside=0.2):
    return gen.random_rays(seed, n, radius=3.0, spread=1.2, inside_frac=inside).astype(np.float64)


def _axis_rays():
    out = []
    for k in range(3):
        for s in (1.0, -1.0):
            o = np.array([0.13, -0.37, 0.29])
            o[k] = -3.0 * s
            d = np.zeros(3)
            d[k] = s
            out.append(np.concatenate([o, d]))
    return np.array(out)


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_recursive_equals_brute_force(oracle_mod, seed):
    t = gen.scene_random(seed, depth=4, sh_degree=1)
    ot = oracle_mod.OracleTree(t)
    rays = np.concatenate([_rays(seed, 300), _axis_rays()])
    for r in rays:
        l0, a0, b0, _ = oracle_mod.trace_ray(ot, r, mode=0)
        l1, a1, b1, _ = oracle_mod.trace_ray(ot, r, mode=1)
        assert np.array_equal(l0, l1)
        np.testing.assert_allclose(a0, a1, atol=1e-12)
        np.testing.assert_allclose(b0, b1, atol=1e-12)


def _dda(o, d, depth, cell_to_leaf, lo=-1.0, edge=2.0):
    """Amanatides & Woo grid stepping over the 2^D grid; returns [(leaf, t_in, t_out)] for occupied cells."""
    G = 1 << depth
    h = edge / G
    d = d / np.linalg.norm(d)
    ch = slab_chord(o, d, lo, lo + edge)
    if ch is None:
        return []
    tn, tf = ch
    p = o + d * (tn + 1e-9 * 0)  # entry point
    # cell of the midpoint of the first tiny step, robust at the entry face
    pm = o + d * (tn + min(1e-7, (tf - tn) * 0.5))
    c = np.clip(np.floor((pm - lo) / h).astype(int), 0, G - 1)
    step = np.sign(d).astype(int)
    tmax = np.empty(3)
    tdel = np.empty(3)
    for k in range(3):
        if d[k] > 0:
            tmax[k] = (lo + (c[k] + 1) * h - o[k]) / d[k]
            tdel[k] = h / d[k]
        elif d[k] < 0:
            tmax[k] = (lo + c[k] * h - o[k]) / d[k]
            tdel[k] = -h / d[k]
        else:
            tmax[k] = np.inf
            tdel[k] = np.inf
    out = []
    t = tn
    while True:
        k = int(np.argmin(tmax))
        t_exit = min(tmax[k], tf)
        leaf = cell_to_leaf.get(tuple(c))
        if leaf is not None and t_exit > t:
            out.append((leaf, t, t_exit))
        if tmax[k] >= tf:
            break
        t = tmax[k]
        c[k] += step[k]
        tmax[k] += tdel[k]
        if c[k] < 0 or c[k] >= G:
            break
    return out


@pytest.mark.parametrize("depth,frac,seed", [(3, 1.0, 0), (4, 0.3, 1), (5, 0.1, 2)])
def test_single_depth_tree_equals_dense_dda(oracle_mod, depth, frac, seed):
    g = rng(seed)
    G = 1 << depth
    allc = np.stack(np.meshgrid(*[np.arange(G)] * 3, indexing="ij"), -1).reshape(-1, 3)
    cells = allc[g.random(allc.shape[0]) < frac]
    child, order = gen.build_from_leaf_cells(cells, depth)
    cells = cells[order]
    n = cells.shape[0]
    t = gen.Tree(depth, np.array([-1, -1, -1], np.float32), 2.0, 0, child, np.ones(n, np.float32),
                 np.zeros((n, 1, 3), np.float32))
    ot = oracle_mod.OracleTree(t)
    c2l = {tuple(c): i for i, c in enumerate(cells)}
    rays = np.concatenate([_rays(seed + 10, 200), _axis_rays()])
    for r in rays:
        ref = _dda(r[:3], r[3:], depth, c2l)
        l0, a0, b0, _ = oracle_mod.trace_ray(ot, r)
        # DDA visits whole cells; merge nothing (one leaf per cell at single depth)
        assert [x[0] for x in ref] == list(l0)
        if len(ref):
            np.testing.assert_allclose([x[1] for x in ref], a0, atol=1e-9)
            np.testing.assert_allclose([x[2] for x in ref], b0, atol=1e-9)


def _locate(child, depth, x, lo=-1.0, edge=2.0):
    """Independent point location: walk the child table with half-open cells."""
    u = (np.asarray(x) - lo) / edge
    node = 0
    for L in range(depth):
        bits = np.floor(u * (1 << (L + 1))).astype(int) & 1
        o = 4 * bits[0] + 2 * bits[1] + bits[2]
        e = int(child[node, o])
        tag, idx = e >> 30, e & ((1 << 30) - 1)
        if tag == 0:
            return None
        if tag == 2:
            return idx
        node = idx
    return None


@pytest.mark.parametrize("seed", [7, 8])
def test_midpoint_query_matches_segment_leaf(oracle_mod, seed):
    t = gen.scene_random(seed, depth=5, sh_degree=0)
    ot = oracle_mod.OracleTree(t)
    for r in _rays(seed, 200):
        leaves, a, b, _ = oracle_mod.trace_ray(ot, r)
        d = r[3:] / np.linalg.norm(r[3:])
        for lf, ta, tb in zip(leaves, a, b):
            assert _locate(t.child, t.depth, r[:3] + d * (0.5 * (ta + tb))) == lf
        # consecutive segments do not overlap and are ordered
        assert np.all(a[1:] >= b[:-1] - 1e-12)


@pytest.mark.parametrize("depth", [1, 2, 4])
def test_full_tree_deltas_sum_to_chord(oracle_mod, depth):
    child, cells = gen.uniform_tree(depth)
    n = cells.shape[0]
    t = gen.Tree(depth, np.array([-1, -1, -1], np.float32), 2.0, 0, child, np.ones(n, np.float32),
                 np.zeros((n, 1, 3), np.float32))
    ot = oracle_mod.OracleTree(t)
    for r in _rays(depth, 100, inside=0.3):
        ch = slab_chord(r[:3], r[3:])
        leaves, a, b, _ = oracle_mod.trace_ray(ot, r)
        if ch is None:
            assert len(leaves) == 0
        else:
            assert abs((b - a).sum() - (ch[1] - ch[0])) < 1e-12


def test_tie_flags_detect_constructed_ties(oracle_mod):
    t = gen.scene_random(3, depth=4, sh_degree=0)
    ot = oracle_mod.OracleTree(t)
    d = np.array([1.0, 1.0, 0.0]) / np.sqrt(2)
    edge_ray = np.concatenate([[-3.0, -3.0, 0.3], d])            # crosses x and y planes together
    clean = np.array([-3.0, 0.1037, 0.2113, 1.0, 0.0123, 0.0371])
    f = oracle_mod.tie_flags(ot, np.stack([edge_ray, clean]))
    assert f[0] & 1 and f[1] == 0

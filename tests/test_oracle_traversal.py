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


def _octant0_tree():
    """Depth 2 in [-1,1]^3: root octant 0 ([-1,0)^3) holds 8 leaves (sigma~ 2), the other 7
    octants are empty boxes."""
    from conftest import make_tree
    L, I = 2 << 30, 1 << 30
    child = [[I | 1] + [0] * 7, [L | k for k in range(8)]]
    return make_tree(child, np.full(8, 2.0), np.zeros((8, 1, 3)), 2, 0)


def test_tie_bit0_only_where_a_leaf_touches_the_crossing(oracle_mod):
    """Reading Q27 (i): a ray along the x = y diagonal crosses an x plane and a y plane at the same
    t at every plane.  At z = 0.3 every cell around those crossings is empty (no leaf can be
    entered or skipped: not a tie); at z = -0.3 the crossings at (-0.5, -0.5) and (0, 0) touch
    the leaves of octant 0 (a tie)."""
    ot = oracle_mod.OracleTree(_octant0_tree())
    d = np.array([1.0, 1.0, 0.0]) / np.sqrt(2)
    empty = np.concatenate([[-3.0, -3.0, 0.3], d])
    leafy = np.concatenate([[-3.0, -3.0, -0.3], d])
    clean = np.array([-3.0, -0.6037, -0.2113, 1.0, 0.0123, 0.0371])
    f = oracle_mod.tie_flags(ot, np.stack([empty, leafy, clean]), gamma=0.0)
    assert f[0] == 0 and f[1] & 1 and f[2] == 0


def test_tie_bit1_sliver_segment(oracle_mod):
    """A ray 1e-9 off the edge x = y = -0.5 (inside octant 0's leaves) cuts a sliver of length
    ~3e-9 out of one leaf: shorter than the fp32 error of its two ends."""
    ot = oracle_mod.OracleTree(_octant0_tree())
    d = np.array([1.0, 1.0, 0.0]) / np.sqrt(2)
    r = np.concatenate([[-3.0, -3.0 + 2e-9, -0.3], d])
    leaves, a, b, _ = oracle_mod.trace_ray(ot, r)
    assert (b - a).min() < 1e-8      # the sliver is really there
    f = oracle_mod.tie_flags(ot, r[None], gamma=0.0)
    assert f[0] & 2


def test_tie_bit2_transmittance_at_gamma_and_bound(oracle_mod):
    """Full depth-1 tree, a ray along +x at y = -0.37, z = 0.21 crosses two unit-length leaves:
    T_1 = exp(-sigma).  sigma = ln(1/gamma) puts T_1 on gamma (a tie; the bound then allows a
    termination flip: >= gamma); sigma = 1 keeps T far from gamma (no tie, bound = the optical
    depth error only)."""
    from conftest import full_depth1
    gamma = 0.01
    r = np.array([[-3.0, -0.37, 0.21, 1.0, 0.0, 0.0]])
    t_tie = oracle_mod.OracleTree(full_depth1(np.log(1.0 / gamma)))
    f, b = oracle_mod.tie_flags(t_tie, r, gamma=gamma, with_bound=True)
    assert f[0] == 4 and b[0] >= gamma
    t_ok = oracle_mod.OracleTree(full_depth1(1.0))
    f, b = oracle_mod.tie_flags(t_ok, r, gamma=gamma, with_bound=True)
    assert f[0] == 0 and 0 < b[0] < 3e-5


def test_tie_bit3_origin_on_a_plane(oracle_mod):
    from conftest import full_depth1
    ot = oracle_mod.OracleTree(full_depth1(1.0))
    on = np.array([0.0, 0.13, 0.21, 0.3, 0.5, 0.7])
    off = np.array([0.013, 0.13, 0.21, 0.3, 0.5, 0.7])
    f = oracle_mod.tie_flags(ot, np.stack([on, off]), gamma=0.0)
    assert f[0] & 8 and not (f[1] & 8)


@pytest.mark.parametrize("which", ["random", "c0"])
def test_tie_bound_covers_rounding_of_the_ray(oracle_mod, c0_tree, which):
    """The per-ray bound of reading Q27 holds for the oracle itself: rendering each ray rounded
    to fp32 (a perturbation of the size any fp32 implementation sees) instead of the double ray
    changes C by at most the bound of the tie rays (+ 1e-5 for the smooth change of tie-free
    rays), and tie-free rays keep their leaf sequence."""
    if which == "c0":
        t = c0_tree
        cam, W, H = gen.config_camera("c0")
        rays = oracle_mod.camera_rays(cam, W, H)
    else:
        t = gen.scene_random(77, depth=5, sh_degree=1, sigma_scale=20.0)
        rays = _rays(78, 3000)
    ot = oracle_mod.OracleTree(t)
    r32 = rays.astype(np.float32).astype(np.float64)
    for gamma in (0.01, 0.0):
        f, b = oracle_mod.tie_flags(ot, rays, gamma=max(gamma, 1e-30), with_bound=True)
        a = oracle_mod.render(ot, rays, gamma=gamma, max_leaves=128)
        c = oracle_mod.render(ot, r32, gamma=gamma, max_leaves=128)
        diff = np.abs(a["rgb"] - c["rgb"]).max(axis=1)
        assert np.all(diff <= b + 1e-5)
        ok = f == 0
        assert np.array_equal(a["leaf_ids"][ok], c["leaf_ids"][ok])

"""Pins for the oracle's NEXT rows: f4 alpha / expected-depth maps (P:468 alpha maps, P:638
depth map; reading Q34) and f1 visibility filtering, the per-leaf maximum ray weight
1 - exp(-sigma_i delta_i) (reading Q33).  Checked against geometric-series closed
forms on uniform rows of cells, Beer-Lambert chords, the early-stop count and an independent
point-location walk -- not against the oracle's own traversal."""
import math

import numpy as np
import pytest

import gen
from conftest import full_depth1, make_tree, slab_chord
from test_oracle_traversal import _locate


def _uniform(depth, sigma):
    child, cells = gen.uniform_tree(depth)
    n = cells.shape[0]
    return make_tree(child, np.full(n, sigma, np.float32), np.zeros((n, 1, 3)), depth, 0), child


def _row_closed_form(t_a, h, sig, N):
    """sum_{i<N} w_i (t_a + (i + 1/2) h) with w_i = q^i (1 - q), q = e^{-sig h}: geometric series."""
    q = math.exp(-sig * h)
    s0 = (1 - q ** N) / (1 - q)                                   # sum q^i
    s1 = q * (1 - N * q ** (N - 1) + (N - 1) * q ** N) / (1 - q) ** 2   # sum i q^i
    return (1 - q) * ((t_a + 0.5 * h) * s0 + h * s1), 1 - q ** N


@pytest.mark.parametrize("depth,sig", [(2, 0.3), (3, 1.7), (4, 0.05)])
def test_depth_alpha_row_closed_form(oracle_mod, depth, sig):
    om = oracle_mod
    t, _ = _uniform(depth, sig)
    sig32 = float(np.float32(sig))
    G = 1 << depth
    h = 2.0 / G
    # axis ray along +x through cell interiors, starting 0.75 before the box
    ray = np.array([[-1.75, -1 + 0.37 * h, -1 + 1.61 * h, 1.0, 0.0, 0.0]])
    a, d = om.render_depth(om.OracleTree(t), ray, gamma=0.0)
    want_d, want_a = _row_closed_form(0.75, h, sig32, G)
    assert abs(d[0] - want_d) < 1e-12 * max(1.0, want_d)
    assert abs(a[0] - want_a) < 1e-13


def test_depth_stops_with_the_ray(oracle_mod):
    """With gamma the sums stop after the segment where T first drops below gamma (Q11)."""
    om = oracle_mod
    depth, sig, gamma = 4, 3.0, 0.05
    t, _ = _uniform(depth, sig)
    sig32 = float(np.float32(sig))
    h = 2.0 / (1 << depth)
    m = next(i + 1 for i in range(1 << depth) if math.exp(-sig32 * h * (i + 1)) < gamma)
    ray = np.array([[-1.5, -1 + 0.41 * h, -1 + 2.33 * h, 1.0, 0.0, 0.0]])
    a, d = om.render_depth(om.OracleTree(t), ray, gamma=gamma)
    want_d, want_a = _row_closed_form(0.5, h, sig32, m)
    assert abs(d[0] - want_d) < 1e-12 and abs(a[0] - want_a) < 1e-13


def test_alpha_is_beer_lambert_and_empty_is_zero(oracle_mod):
    om = oracle_mod
    t, _ = _uniform(3, 0.9)
    rays = gen.random_rays(5, 60, inside_frac=0.3).astype(np.float64)
    a, d = om.render_depth(om.OracleTree(t), rays, gamma=0.0)
    for r, ai, di in zip(rays, a, d):
        ch = slab_chord(r[:3], r[3:])
        want = 0.0 if ch is None else 1 - math.exp(-float(np.float32(0.9)) * (ch[1] - ch[0]))
        assert abs(ai - want) < 1e-13
        if ch is not None:   # expected depth of a constant medium lies inside the chord
            assert ch[0] * ai - 1e-12 <= di <= ch[1] * ai + 1e-12
    t0, _ = _uniform(2, -1.0)   # sigma~ <= 0 everywhere: nothing absorbs
    a0, d0 = om.render_depth(om.OracleTree(t0), rays, gamma=0.0)
    assert not a0.any() and not d0.any()


def test_max_alpha_row_with_early_stop(oracle_mod):
    """One +x ray through a uniform row: the first m cells (the terminating one included, Q11)
    get 1 - e^{-sigma h}; every other leaf keeps 0.  Leaves found by an independent walk."""
    om = oracle_mod
    depth, sig, gamma = 3, 2.0, 0.1
    t, child = _uniform(depth, sig)
    sig32 = float(np.float32(sig))
    G = 1 << depth
    h = 2.0 / G
    m = next(i + 1 for i in range(G) if math.exp(-sig32 * h * (i + 1)) < gamma)
    y, z = -1 + 4.3 * h, -1 + 6.6 * h
    ray = np.array([[-1.2, y, z, 1.0, 0.0, 0.0]])
    got = om.leaf_max_alpha(om.OracleTree(t), ray, gamma=gamma)
    want = np.zeros(t.sigma.shape[0])
    for i in range(m):
        want[_locate(child, depth, [-1 + (i + 0.5) * h, y, z])] = 1 - math.exp(-sig32 * h)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-15)
    # a maximum, not a sum: repeating the ray changes nothing; gamma = 0 reaches the whole row
    np.testing.assert_array_equal(om.leaf_max_alpha(om.OracleTree(t), np.repeat(ray, 3, 0), gamma=gamma), got)
    assert (om.leaf_max_alpha(om.OracleTree(t), ray, gamma=0.0) > 0).sum() == G


def test_max_alpha_diagonal_chord(oracle_mod):
    """Main-diagonal ray through a depth-1 tree: octants 0 and 7 see chord sqrt(3) (edge 1),
    the others meet it in a point (zero length, Q8) and keep 0; a second, axis ray through
    octant 0 has a shorter chord and does not lower its maximum."""
    om = oracle_mod
    t = full_depth1(0.8)
    s = float(np.float32(0.8))
    rays = np.array([[-2.0, -2.0, -2.0, 1.0, 1.0, 1.0], [-3.0, -0.5, -0.5, 1.0, 0.0, 0.0]])
    got = om.leaf_max_alpha(om.OracleTree(t), rays, gamma=0.0)
    want = np.zeros(8)
    want[0] = want[7] = 1 - math.exp(-s * math.sqrt(3.0))
    want[4] = 1 - math.exp(-s * 1.0)   # octant (+x, -y, -z) on the axis ray
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-14)

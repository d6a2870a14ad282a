"""Pins for the oracle's quadrature (Eq. 1-2, background P:864-868,
early stop P:435-437, sigmoid colour Eq. 5) against closed forms and invariants."""
import math

import numpy as np
import pytest

import gen
from conftest import full_depth1, make_tree, rng, slab_chord


def _render(om, tree, rays, **kw):
    return om.render(om.OracleTree(tree), np.atleast_2d(rays), **kw)


def test_sigmoid_zero_coefficients_give_half(oracle_mod):
    # k = 0 -> c = S(0) = 0.5; an opaque slab shows the leaf colour only
    t = full_depth1(200.0, sh_degree=3, k=0.0)
    r = _render(oracle_mod, t, [[-3, 0.1, 0.2, 1, 0, 0]], gamma=0.0, bg=(0, 0, 0))
    np.testing.assert_allclose(r["rgb"][0], 0.5 * (1 - math.exp(-400.0)), atol=1e-15)


def test_beer_lambert_constant_sigma(oracle_mod):
    # constant-sigma region: T = exp(-sigma * chord) for any subdivision (BJ.north_star)
    for depth in (1, 2, 3):
        child, cells = gen.uniform_tree(depth)
        n = cells.shape[0]
        t = make_tree(child, np.full(n, 0.7), np.zeros((n, 1, 3)), depth, 0)
        rays = gen.random_rays(11 + depth, 50, inside_frac=0.3).astype(np.float64)
        res = _render(oracle_mod, t, rays, gamma=0.0)
        for r, T in zip(rays, res["T"]):
            ch = slab_chord(r[:3], r[3:])
            want = 1.0 if ch is None else math.exp(-float(np.float32(0.7)) * (ch[1] - ch[0]))
            assert abs(T - want) < 1e-13


def test_ln2_single_segment(oracle_mod):
    # one segment with sigma*delta = ln 2: w0 = 0.5, T = 0.5, c0 = 0.5 (k = 0)
    child = [[(2 << 30) | 0] + [0] * 7]
    t = make_tree(child, [math.log(2.0)], np.zeros((1, 1, 3)), 1, 0)
    bg = (0.2, 0.4, 0.6)
    r = _render(oracle_mod, t, [[-3, -0.5, -0.5, 1, 0, 0]], gamma=0.0, bg=bg)
    T = math.exp(-float(np.float32(math.log(2.0))))   # sigma is stored as fp32
    assert abs(T - 0.5) < 1e-7 and abs(r["T"][0] - T) < 1e-15
    np.testing.assert_allclose(r["rgb"][0], 0.5 * (1 - T) + T * np.array(bg), atol=1e-15)
    assert r["n_proc"][0] == 1


def test_weights_sum_to_one(oracle_mod):
    # T_N + sum w_i = 1: saturated white leaves (c = 1) on black background give C = 1 - T
    t = gen.scene_random(21, depth=4, sh_degree=0)
    sh = np.zeros_like(t.sh)
    sh[:, 0, :] = 200.0
    t.sh = sh
    rays = gen.random_rays(22, 300, inside_frac=0.2)
    r = _render(oracle_mod, t, rays, gamma=0.0, bg=(0, 0, 0))
    np.testing.assert_allclose(r["rgb"], np.repeat(1 - r["T"][:, None], 3, 1), atol=1e-13)
    r1 = _render(oracle_mod, t, rays, gamma=0.0, bg=(1, 1, 1))
    np.testing.assert_allclose(r1["rgb"], 1.0, atol=1e-13)


def test_transmittance_monotone_in_sigma(oracle_mod):
    t = gen.scene_random(23, depth=4, sh_degree=1)
    rays = gen.random_rays(24, 200)
    base = _render(oracle_mod, t, rays, gamma=0.0)["T"]
    t2 = gen.scene_random(23, depth=4, sh_degree=1)
    t2.sigma = t2.sigma + np.abs(rng(25).normal(size=t2.sigma.shape)).astype(np.float32)
    more = _render(oracle_mod, t2, rays, gamma=0.0)["T"]
    assert np.all(more <= base + 1e-15)


def test_early_stop_bound(oracle_mod, c0_tree):
    # |C_gamma - C_0| <= gamma per channel -- dropped tail mass <= T_stop < gamma
    ot = oracle_mod.OracleTree(c0_tree)
    cam, W, H = gen.config_camera("c0")
    rays = oracle_mod.camera_rays(cam, W, H)
    a = oracle_mod.render(ot, rays, gamma=0.01)
    b = oracle_mod.render(ot, rays, gamma=0.0)
    assert np.abs(a["rgb"] - b["rgb"]).max() <= 0.01
    assert (a["n_proc"] < b["n_proc"]).sum() > 100   # early stop actually happens on c0


def test_early_stop_placement(oracle_mod):
    # reading Q11: the segment that takes T below gamma is composited, then the ray stops
    child = [[(2 << 30) | 0, 0, 0, 0, (2 << 30) | 1, 0, 0, 0]]
    s0 = -math.log(0.005)                       # T after leaf 0 (delta = 1) = 0.005 < 0.01
    t = make_tree(child, [s0, 5.0], np.zeros((2, 1, 3)), 1, 0)
    r = _render(oracle_mod, t, [[-3, -0.5, -0.5, 1, 0, 0]], gamma=0.01, bg=(0, 0, 0), max_leaves=4)
    assert r["n_proc"][0] == 1 and list(r["leaf_ids"][0]) == [0, -1, -1, -1]
    T = math.exp(-float(np.float32(s0)))
    assert abs(r["T"][0] - T) < 1e-15
    np.testing.assert_allclose(r["rgb"][0], 0.5 * (1 - T), atol=1e-15)
    r0 = _render(oracle_mod, t, [[-3, -0.5, -0.5, 1, 0, 0]], gamma=0.0, bg=(0, 0, 0))
    assert r0["n_proc"][0] == 2


def test_empty_tree_and_misses_give_background(oracle_mod):
    t = make_tree([[0] * 8], np.zeros(0), np.zeros((0, 1, 3)), 3, 0)
    bg = (0.1, 0.7, 0.3)
    rays = gen.random_rays(31, 20, inside_frac=0.5)
    r = _render(oracle_mod, t, rays, bg=bg)
    np.testing.assert_allclose(r["rgb"], np.tile(bg, (20, 1)), atol=0)
    assert np.all(r["T"] == 1.0) and np.all(r["n_proc"] == 0)
    t2 = full_depth1(5.0)
    miss = _render(oracle_mod, t2, [[3, 3, 3, 1, 0, 0], [0, 0, 5, 0, 0, 1]], bg=bg)
    np.testing.assert_allclose(miss["rgb"], np.tile(bg, (2, 1)), atol=0)
    assert np.all(miss["nodes_met"] == 0)


def test_origin_inside_box(oracle_mod):
    # t_near = max(0, entry) (reading Q6): from the box centre along +x the chord is 1
    t = full_depth1(1.0)
    r = _render(oracle_mod, t, [[0.0, 0.3, 0.3, 1, 0, 0]], gamma=0.0)
    assert abs(r["T"][0] - math.exp(-1.0)) < 1e-15

"""Pins for the oracle's analytic derivatives (App. B.3) against
central finite differences of the oracle's own forward, closed forms and invariants.

Metric (reading Q26): per tensor relative L2 <= 1e-3 and per component
|d| <= 1e-3 |ref| + 1e-6 max|ref|.  The oracle meets it with orders of margin.
"""
import math

import numpy as np
import pytest

import gen
from conftest import make_tree, rng


def _loss(om, tree, sigma, sh, rays, g, gamma, bg):
    ot = om.OracleTree(tree, sigma=sigma, sh=sh)
    return float((om.render(ot, rays, gamma=gamma, bg=bg)["rgb"] * g).sum())


def _check(ana, fd, tag):
    ana, fd = np.asarray(ana), np.asarray(fd)
    rel = np.linalg.norm(ana - fd) / max(np.linalg.norm(fd), 1e-300)
    assert rel <= 1e-3, (tag, rel)
    tol = 1e-3 * np.abs(fd) + 1e-6 * np.abs(fd).max()
    assert np.all(np.abs(ana - fd) <= tol), (tag, np.abs(ana - fd).max())


def _fd_suite(om, tree, rays, gamma, seed, n_leaves=30):
    bg = np.array([0.9, 0.6, 0.3])
    g = rng(seed).normal(size=(rays.shape[0], 3))
    ot = om.OracleTree(tree)
    gs, gk = om.backward(ot, rays, g, gamma=gamma, bg=bg)
    fw = om.render(ot, rays, gamma=gamma, bg=bg, max_leaves=256)
    touched = np.unique(fw["leaf_ids"][fw["leaf_ids"] >= 0])
    pick = rng(seed + 1).choice(touched, size=min(n_leaves, touched.size), replace=False)
    sig0 = tree.sigma.astype(np.float64)
    sh0 = tree.sh.astype(np.float64)
    a_s, f_s, a_k, f_k = [], [], [], []
    r = rng(seed + 2)
    for lf in pick:
        p = sig0[lf]
        h = 1e-6 * max(1.0, abs(p))
        if p > 10 * h:
            sp, sm = sig0.copy(), sig0.copy()
            sp[lf] += h
            sm[lf] -= h
            fd = (_loss(om, tree, sp, sh0, rays, g, gamma, bg) - _loss(om, tree, sm, sh0, rays, g, gamma, bg)) / (2 * h)
            a_s.append(gs[lf]); f_s.append(fd)
        for _ in range(2):
            b, ch = r.integers(0, sh0.shape[1]), r.integers(0, 3)
            p = sh0[lf, b, ch]
            h = 1e-6 * max(1.0, abs(p))
            kp, km = sh0.copy(), sh0.copy()
            kp[lf, b, ch] += h
            km[lf, b, ch] -= h
            fd = (_loss(om, tree, sig0, kp, rays, g, gamma, bg) - _loss(om, tree, sig0, km, rays, g, gamma, bg)) / (2 * h)
            a_k.append(gk[lf, b, ch]); f_k.append(fd)
    _check(a_s, f_s, "sigma")
    _check(a_k, f_k, "sh")
    return gs, gk


@pytest.mark.parametrize("gamma", [0.0, 0.01])
def test_fd_c0(oracle_mod, c0_tree, gamma):
    cam, W, H = gen.config_camera("c0")
    rays = oracle_mod.camera_rays(cam, W, H)
    ot = oracle_mod.OracleTree(c0_tree)
    flags = oracle_mod.tie_flags(ot, rays, gamma=max(gamma, 1e-30))
    hit = oracle_mod.render(ot, rays)["n_proc"] > 0
    idx = np.flatnonzero(hit & (flags == 0))
    sub = rays[rng(40).choice(idx, 48, replace=False)]
    _fd_suite(oracle_mod, c0_tree, sub, gamma, 41)


@pytest.mark.parametrize("seed", [51, 52])
def test_fd_random_trees(oracle_mod, seed):
    t = gen.scene_random(seed, depth=4, sh_degree=2)
    rays = gen.random_rays(seed, 40, inside_frac=0.2).astype(np.float64)
    _fd_suite(oracle_mod, t, rays, 0.0, seed + 100, n_leaves=20)


def test_single_segment_sigma_zero_closed_form(oracle_mod):
    # dC/dsigma_0 at sigma -> 0+ equals delta_0 (c_0 - c_N); delta = 1 here
    child = [[(2 << 30) | 0] + [0] * 7]
    k = np.array([[[0.3, -1.2, 2.0]]], np.float32).astype(np.float64)   # stored as fp32
    t = make_tree(child, [1e-12], k, 1, 0)
    bg = np.array([0.2, 0.5, 0.9])
    c0 = 1 / (1 + np.exp(-k[0, 0] * 0.5 / math.sqrt(math.pi)))
    for ch in range(3):
        g = np.zeros((1, 3)); g[0, ch] = 1.0
        gs, _ = oracle_mod.backward(oracle_mod.OracleTree(t), [[-3, -0.5, -0.5, 1, 0, 0]], g, bg=bg)
        assert abs(gs[0] - (c0[ch] - bg[ch])) < 1e-9


def test_color_derivative_is_weight(oracle_mod):
    # dC/dc_i = w_i: with l_max = 0, dL/dk_00 = g w c (1-c) Y_00
    child = [[(2 << 30) | 0, 0, 0, 0, (2 << 30) | 1, 0, 0, 0]]
    k = np.array([[[0.4, 0.1, -0.3]], [[1.0, -2.0, 0.5]]], np.float32).astype(np.float64)
    t = make_tree(child, [0.8, 1.7], k, 1, 0)
    Y0 = 0.5 / math.sqrt(math.pi)
    c = 1 / (1 + np.exp(-k[:, 0, :] * Y0))
    w0 = 1 - math.exp(-float(np.float32(0.8)))
    w1 = math.exp(-float(np.float32(0.8))) * (1 - math.exp(-float(np.float32(1.7))))
    g = np.array([[1.0, -2.0, 0.5]])
    _, gk = oracle_mod.backward(oracle_mod.OracleTree(t), [[-3, -0.5, -0.5, 1, 0, 0]], g)
    np.testing.assert_allclose(gk[0, 0], g[0] * w0 * c[0] * (1 - c[0]) * Y0, rtol=1e-12)
    np.testing.assert_allclose(gk[1, 0], g[0] * w1 * c[1] * (1 - c[1]) * Y0, rtol=1e-12)


def test_scale_bounds_gradient(oracle_mod):
    # the per-component magnitude of the summed terms bounds the sum (triangle inequality)
    t = gen.scene_random(65, depth=4, sh_degree=2)
    rays = gen.random_rays(66, 300)
    g = rng(67).normal(size=(300, 3))
    gs, gk, ss, sk = oracle_mod.backward(oracle_mod.OracleTree(t), rays, g, with_scale=True)
    assert np.all(ss >= np.abs(gs) * (1 - 1e-12)) and np.all(sk >= np.abs(gk) * (1 - 1e-12))
    assert ss.max() > 0 and sk.max() > 0


def test_linear_in_dLdC(oracle_mod):
    t = gen.scene_random(61, depth=4, sh_degree=1)
    ot = oracle_mod.OracleTree(t)
    rays = gen.random_rays(62, 100)
    g1, g2 = rng(63).normal(size=(100, 3)), rng(64).normal(size=(100, 3))
    a = oracle_mod.backward(ot, rays, g1)
    b = oracle_mod.backward(ot, rays, g2)
    c = oracle_mod.backward(ot, rays, 2 * g1 - 3 * g2)
    np.testing.assert_allclose(c[0], 2 * a[0] - 3 * b[0], atol=1e-12)
    np.testing.assert_allclose(c[1], 2 * a[1] - 3 * b[1], atol=1e-12)


def test_zero_after_termination_and_relu(oracle_mod):
    # leaf 1 lies behind an opaque leaf 0 (T < gamma after it): zero gradient;
    # leaf 2 has sigma~ < 0: zero sigma gradient, zero colour gradient (w = 0)
    child = [[(2 << 30) | 0, (2 << 30) | 2, 0, 0, (2 << 30) | 1, 0, 0, 0]]
    t = make_tree(child, [10.0, 3.0, -2.0], rng(70).normal(size=(3, 1, 3)), 1, 0)
    ot = oracle_mod.OracleTree(t)
    g = np.ones((2, 3))
    rays = [[-3, -0.5, -0.5, 1, 0, 0], [-0.5, -0.5, -3, 0, 0, 1]]   # 2nd ray: z-ray through leaf 0 then leaf 2
    gs, gk = oracle_mod.backward(ot, rays, g, gamma=0.01)
    assert gs[1] == 0 and np.all(gk[1] == 0)
    assert gs[2] == 0 and np.all(gk[2] == 0)
    assert gs[0] != 0

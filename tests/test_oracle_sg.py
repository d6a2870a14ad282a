"""Pins for the oracle's spherical-Gaussian basis (NEXT f3: G(d; p, lambda)
= exp(lambda (d . p - 1)), 25 lobes in SG-25): the sphere integral 2 pi (1 - e^{-2 lambda}) /
lambda by exact-in-cos(theta) Gauss-Legendre quadrature, rotation invariance, the lambda -> 0
limit (a view-independent colour through the whole renderer) and the peak value at d = p."""
import math

import numpy as np

import gen
from conftest import make_tree


def _lobes(n, seed):
    g = np.random.default_rng(seed)
    p = g.normal(size=(n, 3))
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    return p, g.uniform(0.5, 30.0, size=n)


def test_sphere_integral(oracle_mod):
    """int_S2 G = 2 pi (1 - e^{-2 lambda}) / lambda for a lobe along +z (in cos(theta) the
    integrand is e^{lambda (x - 1)}; 64-point Gauss-Legendre is exact to 1e-12 here)."""
    x, w = np.polynomial.legendre.leggauss(64)
    phi = (np.arange(16) + 0.5) * 2 * np.pi / 16
    ct, ph = np.meshgrid(x, phi, indexing="ij")
    st = np.sqrt(1 - ct ** 2)
    d = np.stack([st * np.cos(ph), st * np.sin(ph), ct], -1).reshape(-1, 3)
    wt = (w[:, None] * np.full(16, 2 * np.pi / 16)[None]).reshape(-1)
    lam = np.array([0.3, 1.0, 4.0, 11.0])
    G = oracle_mod.sg_basis_n(np.tile([0.0, 0.0, 1.0], (4, 1)), lam, d)
    np.testing.assert_allclose((G * wt[:, None]).sum(0), 2 * np.pi * (1 - np.exp(-2 * lam)) / lam, rtol=1e-10)


def test_rotation_invariance_and_peak(oracle_mod):
    p, lam = _lobes(25, 1)
    g = np.random.default_rng(2)
    d = g.normal(size=(200, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    q, _ = np.linalg.qr(g.normal(size=(3, 3)))   # a random orthogonal matrix
    a = oracle_mod.sg_basis_n(p, lam, d)
    b = oracle_mod.sg_basis_n(p @ q.T, lam, d @ q.T)
    np.testing.assert_allclose(a, b, atol=1e-12)
    np.testing.assert_allclose(np.diag(oracle_mod.sg_basis_n(p, lam, p)), 1.0, atol=1e-14)   # G(p; p) = 1
    np.testing.assert_allclose(oracle_mod.sg_basis_n(p[:1], lam[:1], -p[:1]), math.exp(-2 * lam[0]), rtol=1e-12)
    # axes need not be unit length: p is a direction (reading Q36)
    np.testing.assert_allclose(oracle_mod.sg_basis_n(3.7 * p, lam, d), a, atol=1e-12)


def test_zero_bandwidth_gives_view_independent_colour(oracle_mod):
    """lambda = 0 -> G = 1 for every lobe: the leaf colour is S(sum_b k_b) whatever the ray."""
    child, cells = gen.uniform_tree(2)
    n = cells.shape[0]
    g = np.random.default_rng(4)
    k = g.normal(size=(n, 25, 3))
    t = make_tree(child, np.full(n, 500.0), k, 2, 4)
    p, _ = _lobes(25, 5)
    ot = oracle_mod.OracleTree(t, sg=(p, np.zeros(25)))
    rays = gen.random_rays(6, 50).astype(np.float64)
    res = oracle_mod.render(ot, rays, gamma=0.0, bg=(0, 0, 0))
    first, hit = [], []
    for r in rays:
        leaf, t0, t1, _ = oracle_mod.trace_ray(ot, r)
        # sigma delta > 25 in the first leaf: it alone is opaque (e^-25 ~ 1e-11)
        hit.append(leaf.size > 0 and t1[0] - t0[0] > 0.05)
        first.append(leaf[0] if leaf.size else -1)
    first, hit = np.array(first), np.array(hit)
    assert hit.sum() > 10
    kk = k.astype(np.float32).astype(np.float64)
    want = 1 / (1 + np.exp(-kk[first[hit]].sum(1)))
    np.testing.assert_allclose(res["rgb"][hit], want, atol=1e-9)

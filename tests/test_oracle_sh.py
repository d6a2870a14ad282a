"""Pins for the oracle's SH basis (App. B.1) and colour (Eq. 5).

None of these re-call the oracle's own formula: they use closed forms, the
addition theorem, exact quadrature orthonormality, scipy's complex SH and a
textbook Cartesian table.
"""
import json
import math
import os

import numpy as np
import pytest

from conftest import rng

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "sh_closed_forms.json")))


def _unit(n, seed):
    v = rng(seed).normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def test_y00_constant(oracle_mod):
    Y = oracle_mod.sh_basis_n(0, _unit(100, 1))
    np.testing.assert_allclose(Y[:, 0], GOLD["Y00"]["value"], atol=1e-10)


def test_pole_values(oracle_mod):
    Y = oracle_mod.sh_basis(3, [0.0, 0.0, 1.0])
    b = 0
    for l in range(4):
        for m in range(-l, l + 1):
            want = GOLD["pole_m0"]["values"][l] if m == 0 else 0.0
            assert abs(Y[b] - want) < 1e-10, (l, m, Y[b], want)
            b += 1


def test_addition_theorem(oracle_mod):
    Y = oracle_mod.sh_basis_n(3, _unit(500, 2))
    b = 0
    for l in range(4):
        s = (Y[:, b:b + 2 * l + 1] ** 2).sum(1)
        np.testing.assert_allclose(s, GOLD["band_sums"]["values"][l], rtol=0, atol=1e-12)
        b += 2 * l + 1


def test_orthonormal_exact_quadrature(oracle_mod):
    # Gauss-Legendre in cos(theta) x uniform phi is exact for band-limited products (l <= 6 here)
    x, w = np.polynomial.legendre.leggauss(16)
    phi = (np.arange(32) + 0.5) * 2 * np.pi / 32
    ct, ph = np.meshgrid(x, phi, indexing="ij")
    st = np.sqrt(1 - ct ** 2)
    d = np.stack([st * np.cos(ph), st * np.sin(ph), ct], -1).reshape(-1, 3)
    wt = (w[:, None] * np.full(32, 2 * np.pi / 32)[None]).reshape(-1)
    for lmax in (1, 3, 4):
        Y = oracle_mod.sh_basis_n(lmax, d)
        G = (Y * wt[:, None]).T @ Y
        np.testing.assert_allclose(G, np.eye(Y.shape[1]), atol=1e-12)


def test_orthonormal_monte_carlo(oracle_mod):
    # within 5e-3 at >= 1e6 uniform samples
    d = _unit(1_000_000, 3)
    Y = oracle_mod.sh_basis_n(3, d)
    G = 4 * np.pi * (Y.T @ Y) / d.shape[0]
    assert np.abs(G - np.eye(16)).max() < 5e-3


def test_scipy_complex_cross_check(oracle_mod):
    sp = pytest.importorskip("scipy.special")
    d = _unit(64, 4)
    theta = np.arccos(np.clip(d[:, 2], -1, 1))
    phi = np.arctan2(d[:, 1], d[:, 0])
    Y = oracle_mod.sh_basis_n(4, d)
    b = 0
    for l in range(5):   # l = 4: SH-25, the paper's T&T setting
        for m in range(-l, l + 1):
            am = abs(m)
            Yc = sp.sph_harm_y(l, am, theta, phi)   # complex SH, Condon-Shortley phase included
            if m == 0:
                want = Yc.real
            elif m > 0:
                want = math.sqrt(2) * (-1) ** m * Yc.real
            else:
                want = math.sqrt(2) * (-1) ** m * Yc.imag
            np.testing.assert_allclose(Y[:, b], want, atol=1e-12, err_msg=f"l={l} m={m}")
            b += 1


def _textbook_table(d):
    """Cartesian real SH, l <= 3 (the sign-free table that the CS-phase reading of P:755-767 yields)."""
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    pi = np.pi
    c = [
        0.5 * np.sqrt(1 / pi) * np.ones_like(x),
        np.sqrt(3 / (4 * pi)) * y, np.sqrt(3 / (4 * pi)) * z, np.sqrt(3 / (4 * pi)) * x,
        0.5 * np.sqrt(15 / pi) * x * y, 0.5 * np.sqrt(15 / pi) * y * z,
        0.25 * np.sqrt(5 / pi) * (3 * z * z - 1), 0.5 * np.sqrt(15 / pi) * x * z,
        0.25 * np.sqrt(15 / pi) * (x * x - y * y),
        0.25 * np.sqrt(35 / (2 * pi)) * y * (3 * x * x - y * y), 0.5 * np.sqrt(105 / pi) * x * y * z,
        0.25 * np.sqrt(21 / (2 * pi)) * y * (5 * z * z - 1), 0.25 * np.sqrt(7 / pi) * z * (5 * z * z - 3),
        0.25 * np.sqrt(21 / (2 * pi)) * x * (5 * z * z - 1), 0.25 * np.sqrt(105 / pi) * z * (x * x - y * y),
        0.25 * np.sqrt(35 / (2 * pi)) * x * (x * x - 3 * y * y),
    ]
    return np.stack(c, -1)


def test_textbook_cartesian_table(oracle_mod):
    d = _unit(200, 5)
    np.testing.assert_allclose(oracle_mod.sh_basis_n(3, d), _textbook_table(d), atol=1e-12)


def _textbook_l4(d):
    """Cartesian real SH, l = 4, m = -4..4 (same sign-free convention)."""
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    pi = np.pi
    c = [
        0.75 * np.sqrt(35 / pi) * x * y * (x * x - y * y),
        0.75 * np.sqrt(35 / (2 * pi)) * y * z * (3 * x * x - y * y),
        0.75 * np.sqrt(5 / pi) * x * y * (7 * z * z - 1),
        0.75 * np.sqrt(5 / (2 * pi)) * y * z * (7 * z * z - 3),
        3 / 16 * np.sqrt(1 / pi) * (35 * z ** 4 - 30 * z * z + 3),
        0.75 * np.sqrt(5 / (2 * pi)) * x * z * (7 * z * z - 3),
        3 / 8 * np.sqrt(5 / pi) * (x * x - y * y) * (7 * z * z - 1),
        0.75 * np.sqrt(35 / (2 * pi)) * x * z * (x * x - 3 * y * y),
        3 / 16 * np.sqrt(35 / pi) * (x * x * (x * x - 3 * y * y) - y * y * (3 * x * x - y * y)),
    ]
    return np.stack(c, -1)


def test_textbook_cartesian_table_l4(oracle_mod):
    d = _unit(200, 7)
    np.testing.assert_allclose(oracle_mod.sh_basis_n(4, d)[:, 16:], _textbook_l4(d), atol=1e-12)
    # addition theorem for l = 4: sum_m Y_4^m(d)^2 = 9 / (4 pi) for every direction
    np.testing.assert_allclose((oracle_mod.sh_basis_n(4, d)[:, 16:] ** 2).sum(1), 9 / (4 * np.pi), atol=1e-12)


def test_no_cs_convention_flips_odd_m(oracle_mod):
    d = _unit(50, 6)
    a = oracle_mod.sh_basis_n(3, d, cs=1)
    b = oracle_mod.sh_basis_n(3, d, cs=0)
    odd = [1, 3, 5, 7, 9, 11, 13, 15]     # |m| odd, reading Q16
    sign = np.ones(16)
    sign[odd] = -1
    np.testing.assert_allclose(b, a * sign, atol=1e-14)

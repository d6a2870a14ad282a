"""Procedural scenes shaped like the paper's workloads.

SURVEY.md §8(d) fixes the recipes:

* c0 - analytic sphere, 32^3 uniform octree (depth 5), SH degree 1.
* c1 - "NeRF-synthetic-shaped" SDF object (rounded box + sphere + torus with a
  sinusoidal ripple), leaves = depth-9 cells whose centre SDF/h lies in (-3, +1),
  SH degree 3.  The paper's trees hold leaves "at the deepest level while being
  empty elsewhere", which this reproduces.
* c3 - "Tanks&Temples-shaped" bounded scene (ground slab, truck of boxes and
  cylinders, scattered spheres), depth 10, SH degree 3.

The only arithmetic here is the scene SDF and the payload recipe; none of it
is part of the rendering method.
"""
from __future__ import annotations

import hashlib
import os

import numpy as np

from .trees import Tree, build_from_leaf_cells, uniform_tree, random_tree

BBOX_MIN = np.array([-1.0, -1.0, -1.0], dtype=np.float32)
EDGE = 2.0
# amplitude of the l=0 coefficient recipe: +-2.5 in pre-sigmoid colour space
DC_AMPLITUDE = 2.5 * 2.0 * np.sqrt(np.pi)


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=int(seed)))


# ----------------------------------------------------------------------------------------------
# SDF primitives (numpy, float64)
# ----------------------------------------------------------------------------------------------
def _sd_round_box(p, c, b, r):
    q = np.abs(p - c) - (np.asarray(b) - r)
    out = np.linalg.norm(np.maximum(q, 0.0), axis=-1) + np.minimum(q.max(axis=-1), 0.0)
    return out - r


def _sd_sphere(p, c, r):
    return np.linalg.norm(p - c, axis=-1) - r


def _sd_torus_z(p, c, R, r):
    q0 = np.hypot(p[:, 0] - c[0], p[:, 1] - c[1]) - R
    q1 = p[:, 2] - c[2]
    return np.hypot(q0, q1) - r


def _sd_cyl_y(p, c, r, h):
    """Capped cylinder along y: radius r, half-length h."""
    dxz = np.hypot(p[:, 0] - c[0], p[:, 2] - c[2]) - r
    dy = np.abs(p[:, 1] - c[1]) - h
    outside = np.hypot(np.maximum(dxz, 0.0), np.maximum(dy, 0.0))
    return outside + np.minimum(np.maximum(dxz, dy), 0.0)


def sdf_c1(p):
    d = _sd_round_box(p, np.array([0.0, 0.0, -0.55]), (0.8, 0.6, 0.2), 0.05)
    d = np.minimum(d, _sd_sphere(p, np.array([0.0, 0.0, 0.25]), 0.55))
    d = np.minimum(d, _sd_torus_z(p, np.array([0.0, 0.0, 0.1]), 0.75, 0.12))
    return d + 0.015 * np.sin(23 * p[:, 0]) * np.sin(19 * p[:, 1]) * np.sin(17 * p[:, 2])


_C3_SPHERES = None


def _c3_spheres():
    global _C3_SPHERES
    if _C3_SPHERES is None:
        g = _rng(1003)
        n = 14
        ang = g.uniform(0, 2 * np.pi, n)
        rad = g.uniform(0.55, 0.9, n)
        r = g.uniform(0.035, 0.09, n)
        cx, cy = rad * np.cos(ang), rad * np.sin(ang) * 0.95
        cz = -0.65 + r
        _C3_SPHERES = np.stack([cx, cy, cz, r], -1)
    return _C3_SPHERES


def sdf_c3(p):
    d = _sd_round_box(p, np.array([0.0, 0.0, -0.72]), (0.97, 0.97, 0.05), 0.01)          # ground slab
    d = np.minimum(d, _sd_round_box(p, np.array([-0.15, 0.0, -0.36]), (0.42, 0.22, 0.2), 0.03))  # cargo
    d = np.minimum(d, _sd_round_box(p, np.array([0.40, 0.0, -0.42]), (0.14, 0.2, 0.14), 0.04))   # cab
    for x in (-0.45, -0.05, 0.40):
        for y in (-0.23, 0.23):
            d = np.minimum(d, _sd_cyl_y(p, np.array([x, y, -0.58]), 0.085, 0.035))
    for cx, cy, cz, r in _c3_spheres():
        d = np.minimum(d, _sd_sphere(p, np.array([cx, cy, cz]), r))
    return d + 0.004 * np.sin(41 * p[:, 0]) * np.sin(37 * p[:, 1]) * np.sin(43 * p[:, 2])


def shell_cells(sdf, depth: int, lo_h: float = -3.0, hi_h: float = 1.0, lip: float = 1.6,
                start_level: int = 3, chunk: int = 1 << 20):
    """Leaf cells at ``depth`` whose centre SDF / h lies in the open interval (lo_h, hi_h).

    Coarse-to-fine: a level-L cell is refined only if its centre value could
    reach the band given a Lipschitz bound ``lip`` on the SDF.  Chunks are evaluated on a
    thread pool (numpy releases the GIL); the result does not depend on the thread count.
    """
    from concurrent.futures import ThreadPoolExecutor
    h = EDGE / (1 << depth)
    r = np.arange(1 << start_level, dtype=np.int64)
    cells = np.stack(np.meshgrid(r, r, r, indexing="ij"), -1).reshape(-1, 3)
    offs = np.array([[(o >> 2) & 1, (o >> 1) & 1, o & 1] for o in range(8)], dtype=np.int64)
    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as pool:
        for L in range(start_level, depth + 1):
            size = EDGE / (1 << L)

            def keep(c, L=L, size=size):
                centre = BBOX_MIN.astype(np.float64) + (c + 0.5) * size
                f = sdf(centre)
                if L == depth:
                    m = (f / h > lo_h) & (f / h < hi_h)
                else:
                    reach = lip * np.sqrt(3.0) * size * 0.5
                    m = (f - reach < hi_h * h) & (f + reach > lo_h * h)
                return c[m]
            parts = list(pool.map(keep, [cells[s:s + chunk] for s in range(0, cells.shape[0], chunk)]))
            cells = np.concatenate(parts) if parts else np.zeros((0, 3), np.int64)
            if L < depth:
                cells = (cells[:, None, :] * 2 + offs[None]).reshape(-1, 3)
    return cells


# ----------------------------------------------------------------------------------------------
# payload recipes
# ----------------------------------------------------------------------------------------------
def make_payload_random(rng: np.random.Generator, n_leaves: int, sh_degree: int,
                        sigma_scale: float = 4.0, neg_frac: float = 0.1):
    """Generic payload: sigma-tilde ~ |N(0, scale)| with a fraction negated; k ~ N(0, 1)."""
    B = (sh_degree + 1) ** 2
    sigma = np.abs(rng.normal(0.0, sigma_scale, n_leaves))
    neg = rng.random(n_leaves) < neg_frac
    sigma[neg] = -sigma[neg]
    sh = rng.normal(0.0, 1.0, (n_leaves, B, 3))
    return sigma.astype(np.float32), sh.astype(np.float32)


def _payload_c1(rng, cells, depth, sdf_vals, sh_degree=3, sigma_peak=768.0):
    n = cells.shape[0]
    h = EDGE / (1 << depth)
    B = (sh_degree + 1) ** 2
    sigma = sigma_peak / (1.0 + np.exp(2.0 * sdf_vals / h))
    neg = rng.random(n) < 0.05
    sigma[neg] = -np.abs(rng.normal(0.0, 10.0, int(neg.sum())))
    sh = np.empty((n, B, 3), dtype=np.float32)
    omega = np.array([0.021, 0.017, 0.013])
    phase = cells.astype(np.float64) @ omega
    for ch, phi in enumerate((0.0, 2.0, 4.0)):
        sh[:, 0, ch] = DC_AMPLITUDE * np.sin(phase + phi)
    b = 1
    for l in range(1, sh_degree + 1):
        nb = 2 * l + 1
        sh[:, b:b + nb, :] = rng.standard_normal((n, nb, 3), dtype=np.float32) * np.float32(0.8 / (l + 1))
        b += nb
    return sigma.astype(np.float32), sh.astype(np.float32)


# ----------------------------------------------------------------------------------------------
# configs
# ----------------------------------------------------------------------------------------------
def scene_c0(seed: int = 0) -> Tree:
    """c0: sphere r=0.7 at (0.05,-0.03,0.02); uniform depth 5; sigma-tilde 4 inside, -1 outside; SH-1."""
    depth = 5
    child, cells = uniform_tree(depth)
    size = EDGE / (1 << depth)
    centre = BBOX_MIN.astype(np.float64) + (cells + 0.5) * size
    inside = np.linalg.norm(centre - np.array([0.05, -0.03, 0.02]), axis=-1) < 0.7
    sigma = np.where(inside, 4.0, -1.0).astype(np.float32)
    rng = _rng(seed)
    sh = rng.normal(0.0, 1.0, (cells.shape[0], 4, 3)).astype(np.float32)
    return Tree(depth, BBOX_MIN.copy(), EDGE, 1, child, sigma, sh,
                np.full(cells.shape[0], depth, np.int32), cells)


def _source_hash() -> str:
    h = hashlib.sha1()
    here = os.path.dirname(os.path.abspath(__file__))
    for f in ("scenes.py", "trees.py"):
        with open(os.path.join(here, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:12]


def _cached(key: str, build):
    """Disk cache of generated scenes (regenerated whenever missing or when gen/ changes), so
    separate processes (tests, bench, smoke) do not each spend seconds-to-minutes in numpy."""
    d = os.environ.get("PLENOCT_GEN_CACHE", os.path.join(os.path.expanduser("~"), ".cache", "plenoct_gen"))
    path = os.path.join(d, f"{key}_{_source_hash()}.npz")
    if os.path.exists(path):
        try:
            z = np.load(path)
            return Tree(int(z["depth"]), z["bbox_min"], float(z["edge"]), int(z["sh_degree"]), z["child"], z["sigma"],
                        z["sh"], z["leaf_level"], z["leaf_cell"])
        except Exception:
            pass
    t = build()
    try:
        os.makedirs(d, exist_ok=True)
        tmp = path + f".tmp{os.getpid()}.npz"
        np.savez(tmp, depth=t.depth, bbox_min=t.bbox_min, edge=t.edge, sh_degree=t.sh_degree, child=t.child,
                 sigma=t.sigma, sh=t.sh, leaf_level=t.leaf_level, leaf_cell=t.leaf_cell)
        os.replace(tmp, path)
    except Exception:
        pass
    return t


def scene_c1(seed: int = 0, thick: bool = False) -> Tree:
    """c1: NeRF-synthetic-shaped SDF object, depth-9 sparse octree, SH-3, fp32."""
    return _cached(f"c1_s{seed}_t{int(thick)}", lambda: _scene_c1(seed, thick))


def _scene_c1(seed: int, thick: bool) -> Tree:
    depth = 9
    lo = -8.0 if thick else -3.0
    cells = shell_cells(sdf_c1, depth, lo, 1.0)
    child, order = build_from_leaf_cells(cells, depth)
    cells = cells[order]
    size = EDGE / (1 << depth)
    vals = sdf_c1(BBOX_MIN.astype(np.float64) + (cells + 0.5) * size)
    sigma, sh = _payload_c1(_rng(seed), cells, depth, vals, 3)
    return Tree(depth, BBOX_MIN.copy(), EDGE, 3, child, sigma, sh,
                np.full(cells.shape[0], depth, np.int32), cells)


def scene_c3(seed: int = 0, sh_degree: int = 3) -> Tree:
    """c3: Tanks&Temples-shaped bounded scene, depth-10 sparse octree, SH-3 (fp16 payload at upload);
    sh_degree=4 is the paper's own T&T setting, SH-25 (NEXT f3)."""
    key = f"c3_s{seed}" if sh_degree == 3 else f"c3_s{seed}_l{sh_degree}"
    return _cached(key, lambda: _scene_c3(seed, sh_degree))


def _scene_c3(seed: int, sh_degree: int = 3) -> Tree:
    depth = 10
    cells = shell_cells(sdf_c3, depth, -3.0, 1.0)
    child, order = build_from_leaf_cells(cells, depth)
    cells = cells[order]
    size = EDGE / (1 << depth)
    vals = sdf_c3(BBOX_MIN.astype(np.float64) + (cells + 0.5) * size)
    sigma, sh = _payload_c1(_rng(seed), cells, depth, vals, sh_degree, sigma_peak=1536.0)
    return Tree(depth, BBOX_MIN.copy(), EDGE, sh_degree, child, sigma, sh,
                np.full(cells.shape[0], depth, np.int32), cells)


def scene_random(seed: int, depth: int = 4, sh_degree: int = 1, p_split: float = 0.55,
                 p_leaf: float = 0.6, sigma_scale: float = 4.0, bbox_min=(-1.0, -1.0, -1.0),
                 edge: float = 2.0) -> Tree:
    """Tiny random mixed-depth tree (parity / edge cases)."""
    rng = _rng(seed)
    child, lev, cel = random_tree(rng, depth, p_split, p_leaf)
    sigma, sh = make_payload_random(rng, lev.shape[0], sh_degree, sigma_scale)
    return Tree(depth, np.asarray(bbox_min, np.float32), float(edge), sh_degree, child, sigma, sh, lev, cel)

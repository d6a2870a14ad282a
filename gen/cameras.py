"""Cameras and ray batches (inputs only).

Camera record = ``po_camera`` in include/plenoct.h: float32 ``c2w[3][4]`` (camera
to world, OpenGL/Blender axes: x right, y up, -z forward; reading Q5), then
``fx, fy, cx, cy`` in pixels.  16 float32 = 64 bytes.
"""
from __future__ import annotations

import numpy as np

CAMERA_DTYPE = np.dtype([("c2w", np.float32, (3, 4)), ("fx", np.float32), ("fy", np.float32),
                         ("cx", np.float32), ("cy", np.float32)])


def camera_record(c2w: np.ndarray, fx: float, fy: float, cx: float, cy: float) -> np.ndarray:
    rec = np.zeros(1, dtype=CAMERA_DTYPE)
    rec["c2w"][0] = np.asarray(c2w, dtype=np.float64)[:3, :4]
    rec["fx"], rec["fy"], rec["cx"], rec["cy"] = fx, fy, cx, cy
    return rec


def look_at(pos, target=(0.0, 0.0, 0.0), up=(0.0, 0.0, 1.0)) -> np.ndarray:
    pos = np.asarray(pos, np.float64)
    f = np.asarray(target, np.float64) - pos
    f /= np.linalg.norm(f)
    r = np.cross(f, np.asarray(up, np.float64))
    r /= np.linalg.norm(r)
    u = np.cross(r, f)
    c2w = np.zeros((3, 4))
    c2w[:, 0], c2w[:, 1], c2w[:, 2], c2w[:, 3] = r, u, -f, pos
    return c2w


def orbit_camera(radius: float, az_deg: float, el_deg: float, W: int, H: int, focal: float,
                 target=(0.0, 0.0, 0.0)) -> np.ndarray:
    az, el = np.deg2rad(az_deg), np.deg2rad(el_deg)
    pos = np.asarray(target) + radius * np.array([np.cos(el) * np.cos(az), np.cos(el) * np.sin(az), np.sin(el)])
    return camera_record(look_at(pos, target), focal, focal, W / 2.0, H / 2.0)


def config_camera(cfg: str, view: int = 0):
    """Cameras of SURVEY.md §8(d). Returns (camera record, W, H)."""
    if cfg == "c0":
        return orbit_camera(3.0, 23.4, 17.9, 64, 64, 70.0), 64, 64
    if cfg in ("c1", "c2"):
        # c1 view 0 is az 37 deg; the c2 orbit is az = 1.8 deg * i, el 30 deg, radius 3.4
        az = (37.0 if cfg == "c1" else 0.0) + 1.8 * view
        return orbit_camera(3.4, az, 30.0, 800, 800, 1111.111), 800, 800
    if cfg == "c3":
        return orbit_camera(2.6, 20.0 + 1.8 * view, 15.0, 1920, 1080, 1400.0), 1920, 1080
    raise ValueError(cfg)


def fibonacci_hemisphere(n: int, radius: float, W: int, H: int, focal: float) -> np.ndarray:
    """n cameras on the upper hemisphere (Fibonacci lattice), looking at the origin."""
    cams = []
    golden = np.pi * (3.0 - np.sqrt(5.0))
    for i in range(n):
        z = 0.05 + 0.9 * (i + 0.5) / n
        rr = np.sqrt(1.0 - z * z)
        th = golden * i
        pos = radius * np.array([rr * np.cos(th), rr * np.sin(th), z])
        cams.append(camera_record(look_at(pos), focal, focal, W / 2.0, H / 2.0))
    return np.concatenate(cams)


def random_rays(seed: int, n: int, radius: float = 3.0, spread: float = 1.3, inside_frac: float = 0.0):
    """Rays aimed at random points of [-spread, spread]^3 from origins on a sphere of ``radius``.

    A fraction ``inside_frac`` of origins is drawn inside the unit box instead.
    Returns float32 [n][6] = (o, d) with d unit length.
    """
    g = np.random.Generator(np.random.Philox(key=int(seed)))
    v = g.normal(size=(n, 3))
    o = radius * v / np.linalg.norm(v, axis=1, keepdims=True)
    ins = g.random(n) < inside_frac
    o[ins] = g.uniform(-0.95, 0.95, (int(ins.sum()), 3))
    tgt = g.uniform(-spread, spread, (n, 3))
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.concatenate([o, d], axis=1).astype(np.float32)


def camera_rays_f32(cams: np.ndarray, W: int, H: int, view_idx: np.ndarray, pix: np.ndarray) -> np.ndarray:
    """Training-ray batch (config c4 input): pixel-centre rays for (view, pixel) pairs, float32 [n][6]."""
    c = cams[view_idx]
    i = (pix % W).astype(np.float64)
    j = (pix // W).astype(np.float64)
    dc = np.stack([(i + 0.5 - c["cx"]) / c["fx"], -(j + 0.5 - c["cy"]) / c["fy"], -np.ones_like(i)], -1)
    R = c["c2w"][:, :, :3].astype(np.float64)
    d = np.einsum("nij,nj->ni", R, dc)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    o = c["c2w"][:, :, 3].astype(np.float64)
    return np.concatenate([o, d], axis=1).astype(np.float32)

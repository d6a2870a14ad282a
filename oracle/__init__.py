"""CPU oracle for PlenOctree rendering -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_2103_14024_b200``) never imports it and shares no code with it.

It is a ctypes wrapper over ``plenoct_oracle.cpp`` (plain C++17, double
precision, OpenMP over rays), which follows PAPER.md step by step; see the
header of that file for the passages each function restates.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "plenoct_oracle.cpp")
_LIB = os.path.join(_HERE, "libplenoct_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (-O2, -fopenmp, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
                               "-fno-fast-math", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


class OrTree(ctypes.Structure):
    _fields_ = [("child", ctypes.c_void_p), ("n_nodes", ctypes.c_int64), ("sigma", ctypes.c_void_p),
                ("sh", ctypes.c_void_p), ("sh32", ctypes.c_void_p), ("n_leaves", ctypes.c_int64),
                ("depth", ctypes.c_int32),
                ("sh_degree", ctypes.c_int32), ("sh_cs", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("bbox_min", ctypes.c_double * 3), ("edge", ctypes.c_double),
                ("sg_axes", ctypes.c_void_p), ("sg_lambda", ctypes.c_void_p)]


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I64, I32, D = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        _lib.or_sh_basis.argtypes = [ctypes.c_int, ctypes.c_int, P, P]
        _lib.or_sh_basis_n.argtypes = [ctypes.c_int, ctypes.c_int, I64, P, P]
        _lib.or_camera_rays.argtypes = [P, ctypes.c_int, ctypes.c_int, P]
        _lib.or_trace_ray.argtypes = [P, P, ctypes.c_int, I64, P, P, P, P]
        _lib.or_trace_ray.restype = I64
        _lib.or_render.argtypes = [P, P, I64, D, P, ctypes.c_int, P, P, P, I32, P, P, ctypes.c_int]
        _lib.or_backward.argtypes = [P, P, I64, D, P, P, P, P, ctypes.c_int, P, P]
        _lib.or_tie_flags.argtypes = [P, P, I64, D, D, P, P, ctypes.c_int]
        _lib.or_render_depth.argtypes = [P, P, I64, D, P, P, ctypes.c_int]
        _lib.or_leaf_max_alpha.argtypes = [P, P, I64, D, P, ctypes.c_int]
        _lib.or_sg_basis.argtypes = [ctypes.c_int, P, P, I64, P, P]
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


class OracleTree:
    """Holds contiguous copies of the host arrays and the or_tree descriptor."""

    def __init__(self, tree, sh_cs: int = 1, sigma=None, sh=None, sg=None):
        """sg: optional (axes [B][3], lambda [B]) -> spherical-Gaussian basis (NEXT f3)."""
        self.child = np.ascontiguousarray(tree.child, dtype=np.uint32)
        # sigma widened exactly to float64; SH kept as given: float64 arrays (finite-difference
        # tests) are used directly, fp32 / fp16 ones are stored as fp32 and widened exactly in C
        self.sigma = np.ascontiguousarray(tree.sigma if sigma is None else sigma, dtype=np.float64)
        arr = tree.sh if sh is None else sh
        if np.asarray(arr).dtype == np.float64:
            self.sh, self.sh32 = np.ascontiguousarray(arr), None
        else:
            self.sh, self.sh32 = None, np.ascontiguousarray(arr, dtype=np.float32)
        self.B = (tree.sh_degree + 1) ** 2
        self.n_leaves = self.sigma.shape[0]
        self.desc = OrTree(_ptr(self.child).value, self.child.shape[0], _ptr(self.sigma).value,
                           _ptr(self.sh).value if self.sh is not None else None,
                           _ptr(self.sh32).value if self.sh32 is not None else None,
                           self.n_leaves, tree.depth, tree.sh_degree, sh_cs, 0,
                           (ctypes.c_double * 3)(*[float(v) for v in tree.bbox_min]), float(tree.edge),
                           None, None)
        if sg is not None:
            self.sg_axes = np.ascontiguousarray(sg[0], dtype=np.float64).reshape(self.B, 3)
            self.sg_lambda = np.ascontiguousarray(sg[1], dtype=np.float64).reshape(self.B)
            self.desc.sg_axes = _ptr(self.sg_axes).value
            self.desc.sg_lambda = _ptr(self.sg_lambda).value

    @property
    def ref(self):
        return ctypes.byref(self.desc)


def sh_basis(lmax: int, d, cs: int = 1) -> np.ndarray:
    d = np.ascontiguousarray(d, dtype=np.float64)
    Y = np.zeros((lmax + 1) ** 2)
    assert lib().or_sh_basis(lmax, cs, _ptr(d), _ptr(Y)) == 0
    return Y


def sg_basis_n(axes, lam, dirs) -> np.ndarray:
    """Spherical Gaussians G_b(d) = exp(lambda_b (d . p_b - 1)) for dirs [n][3]."""
    axes = np.ascontiguousarray(axes, dtype=np.float64).reshape(-1, 3)
    lam = np.ascontiguousarray(lam, dtype=np.float64).reshape(-1)
    dirs = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
    G = np.zeros((dirs.shape[0], axes.shape[0]))
    assert lib().or_sg_basis(axes.shape[0], _ptr(axes), _ptr(lam), dirs.shape[0], _ptr(dirs), _ptr(G)) == 0
    return G


def sh_basis_n(lmax: int, dirs, cs: int = 1) -> np.ndarray:
    dirs = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
    Y = np.zeros((dirs.shape[0], (lmax + 1) ** 2))
    assert lib().or_sh_basis_n(lmax, cs, dirs.shape[0], _ptr(dirs), _ptr(Y)) == 0
    return Y


def camera_rays(cam_record, W: int, H: int) -> np.ndarray:
    cam = np.ascontiguousarray(np.frombuffer(np.ascontiguousarray(cam_record).tobytes(), dtype=np.float32)[:16])
    rays = np.zeros((H * W, 6))
    lib().or_camera_rays(_ptr(cam), W, H, _ptr(rays))
    return rays


def trace_ray(ot: OracleTree, ray, mode: int = 0, max_seg: int = 4096):
    ray = np.ascontiguousarray(ray, dtype=np.float64)
    leaf = np.zeros(max_seg, np.int64)
    t0 = np.zeros(max_seg)
    t1 = np.zeros(max_seg)
    tnf = np.zeros(2)
    n = lib().or_trace_ray(ot.ref, _ptr(ray), mode, max_seg, _ptr(leaf), _ptr(t0), _ptr(t1), _ptr(tnf))
    n = min(n, max_seg)
    return leaf[:n], t0[:n], t1[:n], tnf


def render(ot: OracleTree, rays, gamma: float = 0.01, bg=(1.0, 1.0, 1.0), mode: int = 0, max_leaves: int = 0,
           nthreads: int = 0):
    """Returns dict(rgb [n,3], T [n], n_proc [n], nodes_met [n], leaf_ids [n,max_leaves] or None)."""
    rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 6)
    n = rays.shape[0]
    bg = np.ascontiguousarray(bg, dtype=np.float64)
    rgb = np.zeros((n, 3))
    T = np.zeros(n)
    n_proc = np.zeros(n, np.int32)
    nodes = np.zeros(n, np.int32)
    ids = np.zeros((n, max_leaves), np.int32) if max_leaves > 0 else None
    lib().or_render(ot.ref, _ptr(rays), n, gamma, _ptr(bg), mode, _ptr(rgb), _ptr(T), _ptr(n_proc), max_leaves,
                    _ptr(ids), _ptr(nodes), nthreads)
    return dict(rgb=rgb, T=T, n_proc=n_proc, nodes_met=nodes, leaf_ids=ids)


def render_depth(ot: OracleTree, rays, gamma: float = 0.01, nthreads: int = 0):
    """NEXT f4: (alpha [n], depth [n]) = (1 - T_stop, sum_i w_i (t_in + t_out) / 2), reading Q34."""
    rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 6)
    a = np.zeros(rays.shape[0])
    d = np.zeros(rays.shape[0])
    lib().or_render_depth(ot.ref, _ptr(rays), rays.shape[0], gamma, _ptr(a), _ptr(d), nthreads)
    return a, d


def leaf_max_alpha(ot: OracleTree, rays, gamma: float = 0.01, nthreads: int = 0) -> np.ndarray:
    """NEXT f1: per-leaf max over rays of 1 - exp(-sigma delta), reading Q33."""
    rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 6)
    m = np.zeros(ot.n_leaves)
    lib().or_leaf_max_alpha(ot.ref, _ptr(rays), rays.shape[0], gamma, _ptr(m), nthreads)
    return m


def backward(ot: OracleTree, rays, dL_dC, gamma: float = 0.0, bg=(1.0, 1.0, 1.0), nthreads: int = 0,
             with_scale: bool = False):
    """Returns (grad_sigma [n_leaves], grad_sh [n_leaves, B, 3]) in float64; with_scale also
    returns the per-component magnitude of the summed terms (rounding-error yardstick)."""
    rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 6)
    g = np.ascontiguousarray(dL_dC, dtype=np.float64).reshape(-1, 3)
    bg = np.ascontiguousarray(bg, dtype=np.float64)
    gs = np.zeros(ot.n_leaves)
    gk = np.zeros((ot.n_leaves, ot.B, 3))
    ss = np.zeros(ot.n_leaves) if with_scale else None
    sk = np.zeros((ot.n_leaves, ot.B, 3)) if with_scale else None
    lib().or_backward(ot.ref, _ptr(rays), rays.shape[0], gamma, _ptr(bg), _ptr(g), _ptr(gs), _ptr(gk), nthreads,
                      _ptr(ss), _ptr(sk))
    return (gs, gk, ss, sk) if with_scale else (gs, gk)


def tie_flags(ot: OracleTree, rays, gamma: float = 0.01, eps: float = 2.0 ** -24, nthreads: int = 0,
              with_bound: bool = False):
    """Tie tags of reading Q27 for an implementation with unit roundoff eps (fp32 by
    default): bit0 an undetermined order of two plane crossings where a leaf touches them, bit1 a
    processed segment within the error of its ends, bit2 T within its error band of gamma before
    the stop, bit3 the origin on a level-D plane.  Every bound is the fp32 error of the crossing
    t = (p - o)/d, evaluated per crossing (plenoct_oracle.cpp, or_tie_flags).  with_bound also
    returns, per ray, the bound on |C_impl - C_oracle| those ties allow (0 for tie-free rays)."""
    rays = np.ascontiguousarray(rays, dtype=np.float64).reshape(-1, 6)
    f = np.zeros(rays.shape[0], np.uint8)
    b = np.zeros(rays.shape[0]) if with_bound else None
    lib().or_tie_flags(ot.ref, _ptr(rays), rays.shape[0], gamma, eps, _ptr(f), _ptr(b), nthreads)
    return (f, b) if with_bound else f

"""B200-native PlenOctree rendering hot path (arXiv 2103.14024): thin Python binding.

Every call marshals arguments to the C ABI of ``libplenoct.so`` (``include/plenoct.h``)
and nothing else: all compute runs in the library's sm_100a CUDA kernels.  PyTorch is
used only for device memory and streams.  If the shared library is missing the import
fails loudly -- there is no CPU fallback.

Names follow the C ABI: ``po_tree_create``, ``po_render``, ``po_render_host``,
``po_render_rays``, ``po_render_backward``, ``po_l2_loss_grad``, ``po_tree_sgd_step``,
``po_trace``, ``po_render_stats``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from ._build import LIB as _LIB_PATH

PO_F32, PO_F16 = 0, 1
PO_SH_CS, PO_SH_NO_CS = 0, 1
PO_TREE_NO_INDEX = 1
STATUS = {0: "PO_OK", 1: "PO_ERR_INVALID_ARG", 2: "PO_ERR_INVALID_TREE", 3: "PO_ERR_OOM", 4: "PO_ERR_CUDA",
          5: "PO_ERR_UNSUPPORTED"}

EXPORTS = ["po_last_error", "po_version", "po_launch_count", "po_tree_create", "po_tree_convert", "po_tree_destroy",
           "po_tree_info", "po_tree_index_bytes", "po_tree_write_leaves", "po_tree_set_sg_basis", "po_tree_leaf_payload",
           "po_tree_read_leaves", "po_render", "po_render_shard", "po_render_host", "po_camera_rays", "po_render_rays", "po_render_rays_ordered",
           "po_render_backward", "po_render_backward_sgd", "po_backward_plan", "po_render_backward_chunk", "po_render_backward_deterministic",
           "po_render_depth", "po_leaf_max_alpha", "po_l2_loss_grad", "po_tree_sgd_step", "po_tree_sgd_step_range", "po_trace", "po_render_stats",
           "po_render_timeline", "po_ray_step_timing", "po_set_block_order"]


class PoError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class TreeDesc(ctypes.Structure):
    _fields_ = [("bbox_min", ctypes.c_float * 3), ("bbox_edge", ctypes.c_float), ("max_depth", ctypes.c_int32),
                ("sh_degree", ctypes.c_int32), ("payload", ctypes.c_int32), ("sh_sign", ctypes.c_int32),
                ("device", ctypes.c_int32), ("flags", ctypes.c_int32)]


class RenderOpts(ctypes.Structure):
    _fields_ = [("gamma", ctypes.c_float), ("background", ctypes.c_float * 3)]


class PoSegments(ctypes.Structure):
    _fields_ = [("records", ctypes.c_void_p), ("count", ctypes.c_void_p), ("n_rays", ctypes.c_int64),
                ("max_seg", ctypes.c_int32)]


class Segments:
    """Caller-owned po_segments buffer (include/plenoct.h): records float32 [max_seg][n][8] and
    count int32 [n] on one device, for the stored-segment pass 2 of a batch of n rays."""

    def __init__(self, n: int, max_seg: int, device=None):
        import torch
        self.n, self.max_seg = int(n), int(max_seg)
        self.records = torch.empty((self.max_seg, self.n, 8), dtype=torch.float32, device=device or "cuda")
        self.count = torch.empty(self.n, dtype=torch.int32, device=self.records.device)

    def struct(self) -> PoSegments:
        return PoSegments(self.records.data_ptr() if self.records.numel() else None, self.count.data_ptr(), self.n,
                          self.max_seg)


def _seg(segments):
    return None if segments is None else ctypes.byref(segments.struct())


_lib = None


def lib():
    """Load libplenoct.so (raises if it has not been built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(_LIB_PATH)
        P, I32, I64, F = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
        L.po_last_error.restype = ctypes.c_char_p
        L.po_version.restype = ctypes.c_char_p
        L.po_launch_count.restype = I64
        L.po_tree_create.argtypes = [P, P, I64, P, P, I64, ctypes.POINTER(P)]
        L.po_tree_destroy.argtypes = [P]
        L.po_tree_convert.argtypes = [P, I32, ctypes.POINTER(P)]
        L.po_tree_write_leaves.argtypes = [P, P, P]
        L.po_tree_set_sg_basis.argtypes = [P, P, P]
        L.po_tree_leaf_payload.argtypes = [P, P, P, P, P]
        L.po_tree_info.argtypes = [P, P, P, P]
        L.po_tree_read_leaves.argtypes = [P, P, P]
        L.po_render.argtypes = [P, P, I32, I32, I32, P, P, P]
        L.po_render_shard.argtypes = [P, P, I32, I32, I32, P, I32, I32, P, P]
        L.po_render_host.argtypes = [P, P, I32, I32, I32, P, P, P]
        L.po_render_rays.argtypes = [P, P, I64, P, P, P, P, P, P]
        L.po_render_rays_ordered.argtypes = [P, P, I64, P, P, P, P, P, P, P]
        L.po_backward_plan.argtypes = [P, P, I64, I32, P, P, P, P, P, P]
        L.po_render_backward_chunk.argtypes = [P, P, P, P, I32, P, P, P, P, P, P, P]
        L.po_camera_rays.argtypes = [P, I32, I32, I32, P, I32, P]
        L.po_render_depth.argtypes = [P, P, I64, P, P, P, P]
        L.po_leaf_max_alpha.argtypes = [P, P, I64, P, P, P]
        L.po_render_backward.argtypes = [P, P, I64, P, P, P, P, P, P, P]
        L.po_render_backward_sgd.argtypes = [P, P, I64, P, P, P, P, F, P, P, P]
        L.po_render_backward_deterministic.argtypes = [P, P, I64, P, P, P, P, P, P, P, P]
        L.po_l2_loss_grad.argtypes = [P, P, I64, P, P, I32, P]
        L.po_tree_sgd_step.argtypes = [P, P, P, F, P]
        L.po_tree_sgd_step_range.argtypes = [P, P, P, F, I64, I64, I32, P]
        L.po_trace.argtypes = [P, P, I64, P, I32, P, P, P, I32, P]
        L.po_tree_index_bytes.argtypes = [P, P]
        L.po_render_stats.argtypes = [P, P, I32, I32, I32, P, P, P]
        L.po_render_timeline.argtypes = [P, P, I32, I32, I32, P, P, P, P]
        L.po_ray_step_timing.argtypes = [P, P, I64, P, I32, P, P, P]
        L.po_set_block_order.argtypes = [P, I32, I32, P]
        for name in EXPORTS:
            if name not in ("po_last_error", "po_version", "po_launch_count"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise PoError(status, lib().po_last_error().decode())


def _ptr(x):
    """Device/host pointer of a torch tensor or numpy array (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, int):   # a raw device address (e.g. an offset view for a shard)
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _opts(gamma: float, background) -> RenderOpts:
    bg = (ctypes.c_float * 3)(*[float(v) for v in background])
    return RenderOpts(float(gamma), bg)


def _need(t, dtype, shape_tail=None, cuda=True):
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch tensor")
    if cuda and not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"expected {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    if shape_tail is not None and tuple(t.shape[-len(shape_tail):]) != tuple(shape_tail):
        raise ValueError(f"expected trailing shape {shape_tail}, got {tuple(t.shape)}")
    return t


class PlenOctree:
    """Owner of a ``po_tree*`` (device copy of the tree)."""

    def __init__(self, handle, desc: TreeDesc, n_nodes: int, n_leaves: int):
        self._h = handle
        self.desc = desc
        self.n_nodes = n_nodes
        self.n_leaves = n_leaves
        self.sh_degree = desc.sh_degree
        self.B = (desc.sh_degree + 1) ** 2
        self.device = desc.device

    @property
    def handle(self):
        if self._h is None:
            raise ValueError("tree destroyed")
        return self._h

    def info(self):
        nn, nl, rb = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
        _check(lib().po_tree_info(self.handle, ctypes.byref(nn), ctypes.byref(nl), ctypes.byref(rb)))
        return nn.value, nl.value, rb.value

    def index_bytes(self) -> int:
        b = ctypes.c_int64()
        _check(lib().po_tree_index_bytes(self.handle, ctypes.byref(b)))
        return b.value

    def read_leaves(self):
        sig = np.zeros(self.n_leaves, np.float32)
        sh = np.zeros((self.n_leaves, self.B, 3), np.float32)
        _check(lib().po_tree_read_leaves(self.handle, _ptr(sig), _ptr(sh)))
        return sig, sh

    def write_leaves(self, sigma, sh):
        sigma = np.ascontiguousarray(sigma, dtype=np.float32).reshape(self.n_leaves)
        sh = np.ascontiguousarray(sh, dtype=np.float32).reshape(self.n_leaves, self.B, 3)
        _check(lib().po_tree_write_leaves(self.handle, _ptr(sigma), _ptr(sh)))

    def set_sg_basis(self, axes=None, lam=None):
        """Spherical-Gaussian basis (B lobes: axes [B][3], bandwidths [B]); None restores SH."""
        if axes is None:
            _check(lib().po_tree_set_sg_basis(self.handle, None, None))
            return
        axes = np.ascontiguousarray(axes, dtype=np.float32).reshape(self.B, 3)
        lam = np.ascontiguousarray(lam, dtype=np.float32).reshape(self.B)
        _check(lib().po_tree_set_sg_basis(self.handle, _ptr(axes), _ptr(lam)))

    def payload_views(self):
        """(sigma [capacity], sh rows [capacity][sh_row]) as torch views of the tree's own fp32
        device arrays (po_tree_leaf_payload); capacity includes the zeroed spare leaves."""
        import torch
        if self.desc.payload != PO_F32:
            raise ValueError("payload views are for fp32 trees")
        sig, sh = ctypes.c_void_p(), ctypes.c_void_p()
        row, cap = ctypes.c_int32(), ctypes.c_int64()
        _check(lib().po_tree_leaf_payload(self.handle, ctypes.byref(sig), ctypes.byref(sh), ctypes.byref(row),
                                          ctypes.byref(cap)))

        class _Dev:   # __cuda_array_interface__ wrapper (torch.as_tensor makes a zero-copy view)
            def __init__(self, ptr, shape):
                self.__cuda_array_interface__ = {"shape": shape, "typestr": "<f4", "data": (ptr, False),
                                                 "version": 3, "strides": None}

        dev = torch.device("cuda", self.device)
        s_t = torch.as_tensor(_Dev(sig.value, (cap.value,)), device=dev)
        k_t = torch.as_tensor(_Dev(sh.value, (cap.value, row.value)), device=dev)
        return s_t, k_t

    def destroy(self):
        if self._h is not None:
            lib().po_tree_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def po_tree_create(child, sigma, sh, depth: int, sh_degree: int, bbox_min=(-1.0, -1.0, -1.0), edge: float = 2.0,
                   payload: int = PO_F32, sh_sign: int = PO_SH_CS, device: int = 0, index: bool = True) -> PlenOctree:
    """Upload a tree from host arrays (child uint32[n_nodes][8], sigma f32[n_leaves], sh f32[n_leaves][B][3]);
    index=False skips the level-(D-1) cell index (PO_TREE_NO_INDEX)."""
    child = np.ascontiguousarray(child, dtype=np.uint32).reshape(-1, 8)
    sigma = np.ascontiguousarray(sigma, dtype=np.float32).reshape(-1)
    B = (sh_degree + 1) ** 2
    sh = np.ascontiguousarray(sh, dtype=np.float32).reshape(sigma.shape[0], B, 3)
    desc = TreeDesc((ctypes.c_float * 3)(*[float(v) for v in bbox_min]), float(edge), int(depth), int(sh_degree),
                    int(payload), int(sh_sign), int(device), 0 if index else PO_TREE_NO_INDEX)
    h = ctypes.c_void_p()
    _check(lib().po_tree_create(ctypes.byref(desc), _ptr(child), child.shape[0], _ptr(sigma), _ptr(sh),
                                sigma.shape[0], ctypes.byref(h)))
    return PlenOctree(h, desc, child.shape[0], sigma.shape[0])


def po_tree_convert(tree: PlenOctree, payload: int = PO_F16) -> PlenOctree:
    """Export a (trained, fp32) tree with another payload, e.g. fp16."""
    h = ctypes.c_void_p()
    _check(lib().po_tree_convert(tree.handle, int(payload), ctypes.byref(h)))
    desc = TreeDesc.from_buffer_copy(tree.desc)
    desc.payload = int(payload)
    return PlenOctree(h, desc, tree.n_nodes, tree.n_leaves)


def tree_from_gen(tree, payload: int = PO_F32, sh_sign: int = PO_SH_CS, device: int = 0,
                  index: bool = True) -> PlenOctree:
    """Upload a ``gen.Tree`` (input-generator output)."""
    return po_tree_create(tree.child, tree.sigma, tree.sh, tree.depth, tree.sh_degree, tree.bbox_min, tree.edge,
                          payload, sh_sign, device, index)


def po_render(tree: PlenOctree, cams, W: int, H: int, out=None, gamma: float = 0.01, background=(1.0, 1.0, 1.0),
              stream=None):
    """cams: CUDA uint8/float32 tensor holding po_camera records ([n][16] float32). Returns [n][H][W][3]."""
    import torch
    cams = _need(cams, torch.float32, (16,))
    n = cams.shape[0]
    if out is None:
        out = torch.empty((n, H, W, 3), dtype=torch.float32, device=cams.device)
    _need(out, torch.float32, (H, W, 3))
    o = _opts(gamma, background)
    _check(lib().po_render(tree.handle, _ptr(cams), n, W, H, ctypes.byref(o), _ptr(out), _stream(stream)))
    return out


def po_render_shard(tree: PlenOctree, cams, W: int, H: int, shard_index: int, shard_count: int, out=None,
                    gamma: float = 0.01, background=(1.0, 1.0, 1.0), stream=None):
    """Render only this shard's 16x16 blocks of the views (others untouched; `out` zeroed if new)."""
    import torch
    cams = _need(cams, torch.float32, (16,))
    n = cams.shape[0]
    if out is None:
        out = torch.zeros((n, H, W, 3), dtype=torch.float32, device=cams.device)
    _need(out, torch.float32, (H, W, 3))
    o = _opts(gamma, background)
    _check(lib().po_render_shard(tree.handle, _ptr(cams), n, W, H, ctypes.byref(o), int(shard_index),
                                 int(shard_count), _ptr(out), _stream(stream)))
    return out


def po_render_host(tree: PlenOctree, cams_host: np.ndarray, W: int, H: int, out_host=None, gamma: float = 0.01,
                   background=(1.0, 1.0, 1.0), stream=None):
    """Host cameras (float32 [n][16]) -> host image (float32 [n][H][W][3], pinned recommended). Synchronous."""
    cams_host = np.ascontiguousarray(np.asarray(cams_host).view(np.float32).reshape(-1, 16))
    n = cams_host.shape[0]
    if out_host is None:
        out_host = np.empty((n, H, W, 3), np.float32)
    o = _opts(gamma, background)
    _check(lib().po_render_host(tree.handle, _ptr(cams_host), n, W, H, ctypes.byref(o), _ptr(out_host),
                                _stream(stream)))
    return out_host


def po_camera_rays(cams, W: int, H: int, stream=None):
    """The exact fp32 rays po_render generates: CUDA float32 [n][H][W][6] (origin, un-normalised d)."""
    import torch
    cams = _need(cams, torch.float32, (16,))
    rays = torch.empty((cams.shape[0], H, W, 6), dtype=torch.float32, device=cams.device)
    _check(lib().po_camera_rays(_ptr(cams), cams.shape[0], W, H, _ptr(rays), cams.device.index or 0,
                                _stream(stream)))
    return rays


def po_render_rays(tree: PlenOctree, rays, out=None, aux=None, gamma: float = 0.01, background=(1.0, 1.0, 1.0),
                   stream=None, leaf_span=None, segments=None, group_order=None):
    """leaf_span: optional int32 [n][2] tensor (the ABI's uint32 pairs; needs aux) for po_backward_plan;
    segments: optional Segments(n, max_seg) written for the stored-segment pass 2 (needs aux);
    group_order: optional int32 [ceil(n/32)] permutation of the 32-ray groups, the order warps
    claim them (po_render_rays_ordered; outputs unchanged)."""
    import torch
    rays = _need(rays, torch.float32, (6,))
    n = rays.shape[0]
    if out is None:
        out = torch.empty((n, 3), dtype=torch.float32, device=rays.device)
    _need(out, torch.float32, (3,))
    if aux is not None:
        _need(aux, torch.float64, (4,))
    if leaf_span is not None:
        _need(leaf_span, torch.int32, (2,))
    o = _opts(gamma, background)
    if group_order is not None:
        _need(group_order, torch.int32)
        if group_order.numel() != (n + 31) // 32:
            raise ValueError("group_order needs ceil(n/32) entries")
        _check(lib().po_render_rays_ordered(tree.handle, _ptr(rays), n, ctypes.byref(o), _ptr(group_order), _ptr(out),
                                            _ptr(aux), _ptr(leaf_span), _seg(segments), _stream(stream)))
        return out
    _check(lib().po_render_rays(tree.handle, _ptr(rays), n, ctypes.byref(o), _ptr(out), _ptr(aux), _ptr(leaf_span),
                                _seg(segments), _stream(stream)))
    return out


def po_backward_plan(tree: PlenOctree, leaf_span, K: int, leaf_bounds=None, perm=None, chunk_ray_end=None,
                     key_quantiles=None, stream=None):
    """Chunk plan for overlapping pass 2 with the gradient allreduce (include/plenoct.h).
    Returns (perm int32 [n], chunk_ray_end int64 [K] on the device, leaf_end list of K ints);
    key_quantiles (optional int64 [K] device tensor) receives balanced bounds for the next plan."""
    import torch
    _need(leaf_span, torch.int32, (2,))
    n = leaf_span.shape[0]
    if perm is None:
        perm = torch.empty(n, dtype=torch.int32, device=leaf_span.device)
    if chunk_ray_end is None:
        chunk_ray_end = torch.empty(K, dtype=torch.int64, device=leaf_span.device)
    _need(perm, torch.int32)
    _need(chunk_ray_end, torch.int64)
    if key_quantiles is not None:
        _need(key_quantiles, torch.int64)
    bounds = None
    if leaf_bounds is not None:
        if len(leaf_bounds) != K:
            raise ValueError("leaf_bounds needs K entries")
        bounds = (ctypes.c_int64 * K)(*[int(b) for b in leaf_bounds])
    leaf_end = (ctypes.c_int64 * K)()
    _check(lib().po_backward_plan(tree.handle, _ptr(leaf_span), n, int(K), bounds, _ptr(perm), _ptr(chunk_ray_end),
                                  leaf_end, _ptr(key_quantiles), _stream(stream)))
    return perm, chunk_ray_end, list(leaf_end)


def po_render_backward_chunk(tree: PlenOctree, rays, perm, chunk_ray_end, chunk: int, dL_dC, grad_sigma, grad_sh,
                             aux=None, gamma: float = 0.0, background=(1.0, 1.0, 1.0), stream=None, segments=None):
    """po_render_backward over chunk `chunk` of a po_backward_plan (accumulates, +=)."""
    import torch
    rays = _need(rays, torch.float32, (6,))
    _need(perm, torch.int32)
    _need(chunk_ray_end, torch.int64)
    if not 0 <= chunk < chunk_ray_end.shape[0]:
        raise ValueError("chunk outside the plan")
    _need(dL_dC, torch.float32, (3,))
    _need(grad_sigma, torch.float32)
    _need(grad_sh, torch.float32, (tree.B, 3))
    if aux is not None:
        _need(aux, torch.float64, (4,))
    o = _opts(gamma, background)
    _check(lib().po_render_backward_chunk(tree.handle, _ptr(rays), _ptr(perm), _ptr(chunk_ray_end), int(chunk),
                                          _ptr(dL_dC), _ptr(aux), _seg(segments), ctypes.byref(o), _ptr(grad_sigma),
                                          _ptr(grad_sh), _stream(stream)))


def po_render_backward(tree: PlenOctree, rays, dL_dC, grad_sigma, grad_sh, aux=None, gamma: float = 0.0,
                       background=(1.0, 1.0, 1.0), stream=None, segments=None):
    """Accumulates (+=) dL/dsigma~ into grad_sigma [n_leaves] and dL/dk into grad_sh [n_leaves][B][3]."""
    import torch
    rays = _need(rays, torch.float32, (6,))
    _need(dL_dC, torch.float32, (3,))
    _need(grad_sigma, torch.float32)
    _need(grad_sh, torch.float32, (tree.B, 3))
    if aux is not None:
        _need(aux, torch.float64, (4,))
    o = _opts(gamma, background)
    _check(lib().po_render_backward(tree.handle, _ptr(rays), rays.shape[0], _ptr(dL_dC), _ptr(aux), _seg(segments),
                                    ctypes.byref(o), _ptr(grad_sigma), _ptr(grad_sh), _stream(stream)))


def po_render_backward_sgd(tree: PlenOctree, rays, dL_dC, lr: float, grad_sigma, grad_sh, aux, segments,
                           gamma: float = 0.0, background=(1.0, 1.0, 1.0), stream=None):
    """a8 + a9 fused for one replica: sigma~ -= lr dL/dsigma~, k -= lr dL/dk in place on the tree.
    grad_sigma / grad_sh are zero scratch for rays that overflowed the stored segments (zero again
    on return); aux and segments come from this batch's po_render_rays (include/plenoct.h)."""
    import torch
    rays = _need(rays, torch.float32, (6,))
    _need(dL_dC, torch.float32, (3,))
    _need(grad_sigma, torch.float32)
    _need(grad_sh, torch.float32, (tree.B, 3))
    _need(aux, torch.float64, (4,))
    o = _opts(gamma, background)
    _check(lib().po_render_backward_sgd(tree.handle, _ptr(rays), rays.shape[0], _ptr(dL_dC), _ptr(aux), _seg(segments),
                                        ctypes.byref(o), float(lr), _ptr(grad_sigma), _ptr(grad_sh), _stream(stream)))


def po_render_depth(tree: PlenOctree, rays, gamma: float = 0.01, alpha=None, depth=None, stream=None):
    """NEXT f4: (alpha [n], depth [n]) maps of explicit rays (include/plenoct.h, reading Q34)."""
    import torch
    rays = _need(rays, torch.float32, (6,))
    n = rays.shape[0]
    if alpha is None:
        alpha = torch.empty(n, dtype=torch.float32, device=rays.device)
    if depth is None:
        depth = torch.empty(n, dtype=torch.float32, device=rays.device)
    _need(alpha, torch.float32)
    _need(depth, torch.float32)
    o = _opts(gamma, (1.0, 1.0, 1.0))
    _check(lib().po_render_depth(tree.handle, _ptr(rays), n, ctypes.byref(o), _ptr(alpha), _ptr(depth),
                                 _stream(stream)))
    return alpha, depth


def po_leaf_max_alpha(tree: PlenOctree, rays, max_alpha=None, gamma: float = 0.01, stream=None):
    """NEXT f1: max-accumulates 1 - exp(-sigma delta) per leaf over the rays (reading Q33)."""
    import torch
    rays = _need(rays, torch.float32, (6,))
    if max_alpha is None:
        max_alpha = torch.zeros(tree.n_leaves, dtype=torch.float32, device=rays.device)
    _need(max_alpha, torch.float32)
    o = _opts(gamma, (1.0, 1.0, 1.0))
    _check(lib().po_leaf_max_alpha(tree.handle, _ptr(rays), rays.shape[0], ctypes.byref(o), _ptr(max_alpha),
                                   _stream(stream)))
    return max_alpha


def po_render_backward_deterministic(tree: PlenOctree, rays, dL_dC, grad_sigma, grad_sh, aux, segments,
                                     gamma: float = 0.0, background=(1.0, 1.0, 1.0), n_overflow=None, stream=None):
    """Order-fixed (bit-reproducible) pass 2 from stored segments; accumulates (+=)."""
    import torch
    rays = _need(rays, torch.float32, (6,))
    _need(dL_dC, torch.float32, (3,))
    _need(grad_sigma, torch.float32)
    _need(grad_sh, torch.float32, (tree.B, 3))
    _need(aux, torch.float64, (4,))
    if n_overflow is not None:
        _need(n_overflow, torch.int32)
    o = _opts(gamma, background)
    _check(lib().po_render_backward_deterministic(tree.handle, _ptr(rays), rays.shape[0], _ptr(dL_dC), _ptr(aux),
                                                  _seg(segments), ctypes.byref(o), _ptr(grad_sigma), _ptr(grad_sh),
                                                  _ptr(n_overflow), _stream(stream)))


def po_l2_loss_grad(pred, target, dL_dC=None, loss=None, stream=None):
    import torch
    _need(pred, torch.float32, (3,))
    _need(target, torch.float32, (3,))
    if dL_dC is None:
        dL_dC = torch.empty_like(pred)
    if loss is not None:
        _need(loss, torch.float64)
    _check(lib().po_l2_loss_grad(_ptr(pred), _ptr(target), pred.shape[0], _ptr(dL_dC), _ptr(loss),
                                 pred.device.index or 0, _stream(stream)))
    return dL_dC


def po_tree_sgd_step(tree: PlenOctree, grad_sigma, grad_sh, lr: float, stream=None):
    _check(lib().po_tree_sgd_step(tree.handle, _ptr(grad_sigma), _ptr(grad_sh), float(lr), _stream(stream)))


PO_SGD_ZERO_GRAD = 1


def po_tree_sgd_step_range(tree: PlenOctree, grad_sigma, grad_sh, lr: float, begin: int, end: int, stream=None,
                           zero_grad: bool = False):
    _check(lib().po_tree_sgd_step_range(tree.handle, _ptr(grad_sigma), _ptr(grad_sh), float(lr), int(begin), int(end),
                                        PO_SGD_ZERO_GRAD if zero_grad else 0, _stream(stream)))


PO_TRACE_CLASSIC = 1


def po_trace(tree: PlenOctree, rays, max_leaves: int = 64, gamma: float = 0.01, with_nodes: bool = True,
             classic: bool = False, stream=None):
    """Returns (leaf_ids int32 [n][max_leaves], counts int32 [n], node_counts int32 [n] or None).
    The ids / counts come from the production traversal (cell index), or from the classic descent
    with classic=True; node counts always from the classic descent."""
    import torch
    rays = _need(rays, torch.float32, (6,))
    n = rays.shape[0]
    dev = rays.device
    ids = torch.empty((n, max_leaves), dtype=torch.int32, device=dev) if max_leaves > 0 else None
    counts = torch.empty(n, dtype=torch.int32, device=dev)
    nodes = torch.empty(n, dtype=torch.int32, device=dev) if with_nodes else None
    o = _opts(gamma, (1.0, 1.0, 1.0))
    _check(lib().po_trace(tree.handle, _ptr(rays), n, ctypes.byref(o), max_leaves, _ptr(ids), _ptr(counts),
                          _ptr(nodes), PO_TRACE_CLASSIC if classic else 0, _stream(stream)))
    return ids, counts, nodes


def po_render_stats(tree: PlenOctree, cams, W: int, H: int, gamma: float = 0.01, stream=None):
    """Traversal counters for one po_render over ``cams`` (see po_render_stats in plenoct.h)."""
    import torch
    cams = _need(cams, torch.float32, (16,))
    ctr = torch.zeros(7, dtype=torch.int64, device=cams.device)
    o = _opts(gamma, (1.0, 1.0, 1.0))
    _check(lib().po_render_stats(tree.handle, _ptr(cams), cams.shape[0], W, H, ctypes.byref(o), _ptr(ctr),
                                 _stream(stream)))
    v = ctr.cpu().tolist()
    return dict(leaf_visits=v[0], sh_rows=v[1], nodes=v[2], hit_rays=v[3], boxes=v[4], leaf_level_boxes=v[5],
                warp_boxes=v[6])


def po_render_timeline(tree: PlenOctree, cams, W: int, H: int, gamma: float = 0.01, background=(1.0, 1.0, 1.0),
                       stream=None):
    """po_render plus one (t_start_ns, t_end_ns, smid<<32|block, view) record per warp tile."""
    import torch
    cams = _need(cams, torch.float32, (16,))
    n = cams.shape[0]
    out = torch.empty((n, H, W, 3), dtype=torch.float32, device=cams.device)
    # one record per warp tile and hand-out position (split blocks take up to 192 extra positions)
    tl = torch.zeros(((((W + 15) // 16) * ((H + 15) // 16) * n + 192) * 8, 4), dtype=torch.int64, device=cams.device)
    o = _opts(gamma, background)
    _check(lib().po_render_timeline(tree.handle, _ptr(cams), n, W, H, ctypes.byref(o), _ptr(out), _ptr(tl),
                                    _stream(stream)))
    return out, tl


def po_set_block_order(tree: PlenOctree, W: int, H: int, order):
    """Diagnostics: replace the block hand-out order of W x H renders (include/plenoct.h)."""
    order = np.ascontiguousarray(order, dtype=np.uint32)
    _check(lib().po_set_block_order(tree.handle, W, H, _ptr(order)))


def po_ray_step_timing(tree: PlenOctree, rays, max_steps: int = 1024, gamma: float = 0.01, stream=None):
    """Measurement: (rec uint32 [n][max_steps][2], steps int32 [n]) -- include/plenoct.h."""
    import torch
    rays = _need(rays, torch.float32, (6,))
    n = rays.shape[0]
    rec = torch.zeros((n, max_steps, 2), dtype=torch.int32, device=rays.device)
    steps = torch.zeros(n, dtype=torch.int32, device=rays.device)
    o = _opts(gamma, (1.0, 1.0, 1.0))
    _check(lib().po_ray_step_timing(tree.handle, _ptr(rays), n, ctypes.byref(o), int(max_steps), _ptr(rec),
                                    _ptr(steps), _stream(stream)))
    return rec, steps


def launch_count() -> int:
    return int(lib().po_launch_count())


def cams_tensor(cam_records, device="cuda"):
    """po_camera records (numpy structured or float32 [n][16]) -> CUDA float32 [n][16]."""
    import torch
    a = np.ascontiguousarray(cam_records)
    a = np.frombuffer(a.tobytes(), dtype=np.float32).reshape(-1, 16).copy()
    return torch.from_numpy(a).to(device)

"""CPU-side checks of the C ABI: the library loads, exports every symbol include/plenoct.h
declares, and rejects malformed trees / arguments before touching the GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def po():
    import __graft_entry__ as g
    g.build()
    import paper_2103_14024_b200 as po
    po.lib()
    return po


def test_header_symbols_exported(po):
    hdr = open(os.path.join(ROOT, "include", "plenoct.h")).read()
    names = set(re.findall(r"\b(po_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 14
    L = ctypes.CDLL(po._LIB_PATH)
    for n in sorted(names):
        assert hasattr(L, n), n
    assert set(po.EXPORTS) == names


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2103_14024_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).lower().replace("no cpu", ""), f


def _desc(po, depth=2, deg=0, payload=0, flags=0):
    return po.TreeDesc((ctypes.c_float * 3)(-1, -1, -1), 2.0, depth, deg, payload, 0, 0, flags)


def _create(po, child, sigma, sh, depth=2, deg=0, payload=0, flags=0):
    child = np.ascontiguousarray(child, np.uint32)
    sigma = np.ascontiguousarray(sigma, np.float32)
    sh = np.ascontiguousarray(sh, np.float32)
    h = ctypes.c_void_p()
    d = _desc(po, depth, deg, payload, flags)
    st = po.lib().po_tree_create(ctypes.byref(d), child.ctypes.data, child.shape[0], sigma.ctypes.data,
                                 sh.ctypes.data, sigma.shape[0], ctypes.byref(h))
    return st, po.lib().po_last_error().decode()


def test_rejects_malformed_trees(po):
    L = 2 << 30
    I = 1 << 30
    ok_sh = np.zeros((2, 1, 3))
    # leaf index out of range
    st, msg = _create(po, [[L | 0, L | 5, 0, 0, 0, 0, 0, 0]], [1, 1], ok_sh, depth=1)
    assert st == 2 and "out of range" in msg
    # leaf referenced twice
    st, msg = _create(po, [[L | 0, L | 0, 0, 0, 0, 0, 0, 0]], [1, 1], ok_sh, depth=1)
    assert st == 2 and "twice" in msg
    # internal node deeper than max_depth allows
    st, msg = _create(po, [[I | 1] + [0] * 7, [L | 0] + [0] * 7], [1], np.zeros((1, 1, 3)), depth=1)
    assert st == 2 and "max_depth" in msg
    # unreachable node
    st, msg = _create(po, [[L | 0] + [0] * 7, [0] * 8], [1], np.zeros((1, 1, 3)), depth=2)
    assert st == 2 and "unreachable" in msg
    # NaN payload
    st, msg = _create(po, [[L | 0] + [0] * 7], [np.nan], np.zeros((1, 1, 3)), depth=1)
    assert st == 2 and "not finite" in msg
    st, msg = _create(po, [[L | 0] + [0] * 7], [1.0], np.full((1, 1, 3), np.inf), depth=1)
    assert st == 2 and "not finite" in msg
    # unsupported degree / bad depth
    st, _ = _create(po, [[0] * 8], [], np.zeros((0, 36, 3)), depth=1, deg=5)
    assert st == 5
    st, _ = _create(po, [[0] * 8], [], np.zeros((0, 1, 3)), depth=0)
    assert st == 1
    # unknown descriptor flags
    st, msg = _create(po, [[0] * 8], [], np.zeros((0, 1, 3)), depth=1, flags=4)
    assert st == 1 and "flags" in msg


def test_rejects_bad_args_without_gpu(po):
    o = po._opts(2.0, (1, 1, 1))   # gamma outside [0,1]
    st = po.lib().po_render_rays(None, None, 1, ctypes.byref(o), None, None, None, None, None)
    assert st == 1
    # chunk plan: NULL tree, bad K
    assert po.lib().po_backward_plan(None, None, 1, 4, None, None, None, None, None, None) == 1
    assert po.lib().po_render_backward_chunk(None, None, None, None, 0, None, None, None, None, None, None, None) == 1
    # NULL tree handles are rejected before any device work, by every entry point
    L = po.lib()
    assert L.po_render_backward_deterministic(None, None, 1, None, None, None, ctypes.byref(o), None, None, None,
                                              None) == 1
    assert L.po_render_depth(None, None, 1, ctypes.byref(o), None, None, None) == 1
    assert L.po_leaf_max_alpha(None, None, 1, ctypes.byref(o), None, None) == 1
    assert L.po_tree_set_sg_basis(None, None, None) == 1
    assert L.po_tree_write_leaves(None, None, None) == 1
    h = ctypes.c_void_p()
    assert L.po_tree_convert(None, 1, ctypes.byref(h)) == 1 and h.value is None
    assert L.po_tree_sgd_step_range(None, None, None, ctypes.c_float(1.0), 0, 1, 0, None) == 1
    # diagnostics exist in every build and are refused unless built with -DPO_DIAG
    assert L.po_ray_step_timing(None, None, 1, ctypes.byref(o), 8, None, None, None) == 5
    assert L.po_render_timeline(None, None, 1, 8, 8, ctypes.byref(o), None, None, None) == 5
    assert L.po_trace(None, None, 1, ctypes.byref(o), 0, None, None, None, 0, None) == 1
    assert L.po_tree_index_bytes(None, None) == 1
    assert L.po_render_backward_sgd(None, None, 1, None, None, None, ctypes.byref(o), ctypes.c_float(1.0), None, None,
                                    None) == 1


def test_c_example_builds(po):
    """examples/render_uniform.c compiles with -Werror against include/plenoct.h alone and links
    libplenoct.so: the boundary needs no CUDA or torch headers (it runs under -m gpu)."""
    from paper_2103_14024_b200 import _build
    assert os.path.exists(_build.build_example())

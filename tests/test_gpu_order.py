"""Cost-ordered block hand-out of single-view renders (DESIGN.md §6.1 v13): the order in which
16x16 blocks are handed out is a schedule only, so an image must not depend on it.  A view
rendered on a stream whose order table was rewritten by other views (costliest block of the
previous frame first) must equal, bit for bit, the same view rendered first on a fresh stream
(centre-out order), through size changes of the table and across multi-view launches."""
import numpy as np
import pytest

import gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()
    import paper_2103_14024_b200 as po
    return po, torch


def test_image_independent_of_adaptive_order(env, c1_tree):
    po, torch = env
    tree = po.tree_from_gen(c1_tree)
    cams = po.cams_tensor(np.concatenate([gen.config_camera("c1", v)[0] for v in (0, 5, 40, 41)]))
    fresh = torch.cuda.Stream()
    with torch.cuda.stream(fresh):   # first single-view render on this stream: centre-out order
        ref = po.po_render(tree, cams[3:4], 800, 800, stream=fresh)
    fresh.synchronize()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for v in (0, 1, 2):          # orders rewritten from views 0, 5, 40
            po.po_render(tree, cams[v:v + 1], 800, 800, stream=s)
        a = po.po_render(tree, cams[3:4], 800, 800, stream=s)
        po.po_render(tree, cams[0:1], 400, 320, stream=s)   # table re-initialised for another size
        po.po_render(tree, cams[0:1], 800, 800, stream=s)   # and back
        b = po.po_render(tree, cams[3:4], 800, 800, stream=s)
        m = po.po_render(tree, cams[2:4], 800, 800, stream=s)   # multi-view: centre-out, table untouched
        c = po.po_render(tree, cams[3:4], 800, 800, stream=s)
    s.synchronize()
    for x in (a, b, m[1:2], c):
        assert torch.equal(x, ref)


def test_host_render_independent_of_zipped_cost_order(env, c1_tree):
    """po_render_host (pinned image written by the kernel over PCIe) uses the zipped cost order;
    its images must equal the device render of the same view bit for bit."""
    po, torch = env
    tree = po.tree_from_gen(c1_tree)
    cams_np = np.concatenate([gen.config_camera("c1", v)[0] for v in (0, 5, 40, 41)])
    cams = po.cams_tensor(cams_np)
    fresh = torch.cuda.Stream()
    with torch.cuda.stream(fresh):
        ref = po.po_render(tree, cams[3:4], 800, 800, stream=fresh)
    fresh.synchronize()
    pinned = torch.empty((1, 800, 800, 3), dtype=torch.float32, pin_memory=True).numpy()
    s = torch.cuda.Stream()
    for v in range(4):
        po.po_render_host(tree, cams_np[v:v + 1], 800, 800, out_host=pinned, stream=s)
    assert np.array_equal(pinned, ref.cpu().numpy())

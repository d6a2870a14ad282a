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


def test_ragged_sizes_and_tiny_images(env):
    """Ragged image sizes (edge blocks partly outside the image, split sub-blocks included) and
    images with fewer blocks than the split count: repeated renders on one stream (cost-ordered,
    split) equal a first render on a fresh stream."""
    po, torch = env
    tree = po.tree_from_gen(gen.scene_c0())
    cam, _, _ = gen.config_camera("c0")
    ct = po.cams_tensor(cam)
    for W, H in ((203, 117), (64, 64), (16, 16), (5, 3), (33, 17)):
        fresh = torch.cuda.Stream()
        with torch.cuda.stream(fresh):
            ref = po.po_render(tree, ct, W, H, stream=fresh)
        fresh.synchronize()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            outs = [po.po_render(tree, ct, W, H, stream=s) for _ in range(4)]
        s.synchronize()
        for x in outs:
            assert torch.equal(x, ref), (W, H)


def test_render_rays_group_order_is_scheduling_only(env):
    """po_render_rays_ordered (pass-1 claim order of 32-ray groups): colours, double totals, leaf
    spans and stored segments equal po_render_rays' bit for bit, for a ragged ray count."""
    po, torch = env
    t = gen.scene_random(11, depth=6, sh_degree=3, sigma_scale=3.0)
    tree = po.tree_from_gen(t)
    rays = torch.from_numpy(gen.random_rays(12, 5000, inside_frac=0.2)).cuda()
    n = rays.shape[0]
    order = torch.from_numpy(np.random.default_rng(3).permutation((n + 31) // 32).astype(np.int32)).cuda()

    def run(go):
        aux = torch.empty((n, 4), dtype=torch.float64, device="cuda")
        span = torch.empty((n, 2), dtype=torch.int32, device="cuda")
        seg = po.Segments(n, 64)
        seg.records.zero_()
        out = po.po_render_rays(tree, rays, aux=aux, gamma=0.0, leaf_span=span, segments=seg, group_order=go)
        return out, aux, span, seg.count, seg.records

    a, b = run(None), run(order)
    for x, y in zip(a, b):
        assert torch.equal(x, y)

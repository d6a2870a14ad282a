"""a1 ray generation: po_camera_rays is the exact IEEE fp32 evaluation of the camera model
(reading Q5), and po_render(cams) == po_render_rays(po_camera_rays(cams)) bit for bit."""
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


def _numpy_rays(cam, W, H):
    """IEEE fp32 evaluation, same operation order as the header documents."""
    f = np.float32
    c = np.frombuffer(np.ascontiguousarray(cam).tobytes(), dtype=np.float32)[:16]
    i = np.arange(W, dtype=np.float32)[None, :].repeat(H, 0)
    j = np.arange(H, dtype=np.float32)[:, None].repeat(W, 1)
    dx = ((i + f(0.5)) - c[14]) / c[12]
    dy = -(((j + f(0.5)) - c[15]) / c[13])
    d = [((c[k * 4] * dx) + (c[k * 4 + 1] * dy)) - c[k * 4 + 2] for k in range(3)]
    o = [np.full_like(dx, c[k * 4 + 3]) for k in range(3)]
    return np.stack(o + d, -1).astype(np.float32)


def test_camera_rays_bit_exact(env):
    po, torch = env
    for cfg in ("c0", "c1"):
        cam, W, H = gen.config_camera(cfg)
        got = po.po_camera_rays(po.cams_tensor(cam), W, H)[0].cpu().numpy()
        want = _numpy_rays(cam, W, H)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), cfg


def test_render_equals_render_rays_of_camera_rays(env, c1_tree):
    """po_render (persistent k_render with tail balancing: paused rays handed to other warps and
    resumed from their pixel, cell and (T, C)) equals po_render_rays of the same camera rays bit
    for bit: one 3-view launch, then single-view launches back to back on one stream (the queue
    and its ready flags are reused across launches) and on a second stream."""
    po, torch = env
    tree = po.tree_from_gen(c1_tree)
    cams = np.concatenate([gen.config_camera("c1", v)[0] for v in range(8)])
    ct = po.cams_tensor(cams)
    rays = po.po_camera_rays(ct, 800, 800).reshape(-1, 6)
    ref = po.po_render_rays(tree, rays).reshape(8, 800, 800, 3)
    img = po.po_render(tree, ct[:3], 800, 800)
    assert torch.equal(img, ref[:3])
    side = torch.cuda.Stream()
    for rep in range(2):
        for v in range(8):
            if rep == 1 and v % 2:
                with torch.cuda.stream(side):
                    one = po.po_render(tree, ct[v:v + 1], 800, 800, stream=side)
                side.synchronize()
            else:
                one = po.po_render(tree, ct[v:v + 1], 800, 800)
            assert torch.equal(one[0], ref[v]), (rep, v)


def test_tile_shards_assemble_the_frame():
    """po_render_shard: the shards' blocks are disjoint, cover the image, and their sum is
    bit-identical to po_render (SURVEY 8(e) single-view latency mode)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import gen
    import paper_2103_14024_b200 as po
    tree = po.tree_from_gen(gen.scene_random(77, depth=5, sh_degree=2, sigma_scale=3.0))
    cams = po.cams_tensor(np.concatenate([gen.orbit_camera(3.0, 10.0 + 50 * i, 20.0, 100, 72, 80.0)
                                          for i in range(2)]))
    full = po.po_render(tree, cams, 100, 72)
    for n in (1, 3, 4):
        parts = [po.po_render_shard(tree, cams, 100, 72, i, n) for i in range(n)]
        written = [(p != 0).any(dim=-1) for p in parts]
        assert int(sum(w.int() for w in written).max()) <= 1          # disjoint
        assert torch.equal(sum(parts), full)                           # exact assembly
    with pytest.raises(po.PoError):
        po.po_render_shard(tree, cams, 100, 72, 3, 3)

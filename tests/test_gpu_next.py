"""GPU parity of the NEXT rows against the pinned oracle:
f4 alpha / expected-depth maps (po_render_depth, reading Q34) and f1 visibility filtering
(po_leaf_max_alpha, reading Q33).  Tie-free rays only (reading Q27); the bars are
the forward's: 1e-4 absolute on alpha and on depth / max(1, |depth|)."""
import numpy as np
import pytest

import gen

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def env(oracle_mod):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()
    import paper_2103_14024_b200 as po
    return po, oracle_mod, torch


def _tie_free(om, ot, rays, gamma):
    return om.tie_flags(ot, rays, gamma=gamma if gamma > 0 else 1e-30) == 0


def _cases():
    return [("c0", 0.01), ("c0", 0.0), ("random", 0.01), ("random", 0.0)]


def _scene(name):
    if name == "c0":
        t = gen.scene_c0()
        cam, W, H = gen.config_camera("c0")
        return t, cam, W, H, None
    t = gen.scene_random(71, depth=6, sh_degree=1, sigma_scale=3.0)
    return t, None, 0, 0, gen.random_rays(72, 4000, inside_frac=0.1).astype(np.float64)


@pytest.mark.parametrize("name,gamma", _cases())
def test_depth_alpha_match_oracle(env, name, gamma):
    po, om, torch = env
    t, cam, W, H, rays = _scene(name)
    ot = om.OracleTree(t)
    if rays is None:
        rays = om.camera_rays(cam, W, H)
    rays = rays[_tie_free(om, ot, rays, gamma)]
    tree = po.tree_from_gen(t)
    a, d = po.po_render_depth(tree, torch.from_numpy(rays.astype(np.float32)).cuda(), gamma=gamma)
    # the oracle sees the fp32 rays the GPU sees
    ra, rd = om.render_depth(ot, rays.astype(np.float32).astype(np.float64), gamma=gamma)
    a, d = a.cpu().numpy(), d.cpu().numpy()
    assert np.abs(a - ra).max() <= TOL
    assert (np.abs(d - rd) / np.maximum(1.0, np.abs(rd))).max() <= TOL
    assert (ra > 0.5).any()   # the case actually hits something


@pytest.mark.parametrize("name,gamma", _cases())
def test_leaf_max_alpha_matches_oracle(env, name, gamma):
    po, om, torch = env
    t, cam, W, H, rays = _scene(name)
    ot = om.OracleTree(t)
    if rays is None:
        rays = om.camera_rays(cam, W, H)
    rays = rays[_tie_free(om, ot, rays, gamma)].astype(np.float32)
    tree = po.tree_from_gen(t)
    r = torch.from_numpy(rays).cuda()
    got = po.po_leaf_max_alpha(tree, r, gamma=gamma).cpu().numpy()
    want = om.leaf_max_alpha(ot, rays.astype(np.float64), gamma=gamma)
    assert np.abs(got - want).max() <= TOL
    assert (want > 0).sum() > 100
    # max-accumulation across calls (several training views): two halves == one pass
    half = rays.shape[0] // 2
    acc = po.po_leaf_max_alpha(tree, r[:half].contiguous(), gamma=gamma)
    po.po_leaf_max_alpha(tree, r[half:].contiguous(), max_alpha=acc, gamma=gamma)
    np.testing.assert_array_equal(acc.cpu().numpy(), got)


def test_c1_depth_and_filter_sampled(env, c1_tree):
    """c1 scale: 20,000 random pixels of view 0 (tie-free, >= 95 %), depth/alpha and the filter
    statistic of the leaves they reach.  Bars: 1e-4 plus the ray's optical-depth error band
    (reading Q27: with sigma up to 768 the fp32 crossings move a segment's optical depth by
    sigma * (e_in + e_out); alpha = 1 - T moves by at most that sum, the expected depth by at
    most t_far times twice it, a leaf's max alpha by at most the largest band of its rays)."""
    po, om, torch = env
    cam, W, H = gen.config_camera("c1", 0)
    g = np.random.default_rng(5)
    pix = g.choice(W * H, 20000, replace=False)
    rays = om.camera_rays(cam, W, H)[pix].astype(np.float32).astype(np.float64)
    ot = om.OracleTree(c1_tree)
    f, band = om.tie_flags(ot, rays, gamma=0.01, with_bound=True)
    ok = f == 0
    assert ok.mean() >= 0.95
    rays, band = rays[ok], band[ok]
    tree = po.tree_from_gen(c1_tree)
    r = torch.from_numpy(rays.astype(np.float32)).cuda()
    a, d = po.po_render_depth(tree, r, gamma=0.01)
    ra, rd = om.render_depth(ot, rays, gamma=0.01)
    assert np.all(np.abs(a.cpu().numpy() - ra) <= TOL + band)
    t_far = np.linalg.norm(rays[:, :3], axis=1) + 2.0 * np.sqrt(3.0)   # beyond any exit of [-1,1]^3
    assert np.all(np.abs(d.cpu().numpy() - rd) <= TOL * np.maximum(1.0, np.abs(rd)) + 2.0 * t_far * band)
    print(f"c1 f4: max |d alpha| {np.abs(a.cpu().numpy() - ra).max():.2e}, band p50 {np.median(band):.1e} "
          f"max {band.max():.1e}")
    got = po.po_leaf_max_alpha(tree, r, gamma=0.01).cpu().numpy()
    want = om.leaf_max_alpha(ot, rays, gamma=0.01)
    assert np.abs(got - want).max() <= TOL + band.max()
    assert ((got > 0) == (want > 0)).mean() > 0.999


def _sg_lobes(B, seed):
    g = np.random.default_rng(seed)
    p = g.normal(size=(B, 3))
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    return p.astype(np.float32), g.uniform(0.5, 20.0, size=B).astype(np.float32)


@pytest.mark.parametrize("deg,gamma", [(4, 0.01), (4, 0.0), (2, 0.01)])
def test_sg_basis_render_and_backward(env, deg, gamma):
    """NEXT f3 SG-25: render and backward with spherical-Gaussian lobes against the
    oracle on the same (fp32) lobes; SH restored afterwards."""
    po, om, torch = env
    t = gen.scene_random(73 + deg, depth=5, sh_degree=deg, sigma_scale=3.0)
    B = (deg + 1) ** 2
    axes, lam = _sg_lobes(B, 9)
    tree = po.tree_from_gen(t)
    tree.set_sg_basis(axes, lam)
    # the oracle normalises in double what the library normalises in fp32 -> hand it the same axes
    ax32 = (axes.astype(np.float64) / np.linalg.norm(axes.astype(np.float64), axis=1, keepdims=True))
    ot = om.OracleTree(t, sg=(ax32, lam.astype(np.float64)))
    rays = gen.random_rays(74, 3000, inside_frac=0.1).astype(np.float64)
    rays = rays[_tie_free(om, ot, rays, gamma)]
    r = torch.from_numpy(rays.astype(np.float32)).cuda()
    out = po.po_render_rays(tree, r, gamma=gamma).cpu().numpy()
    ref = om.render(ot, rays.astype(np.float32).astype(np.float64), gamma=gamma)
    assert np.abs(out - ref["rgb"]).max() <= TOL
    g = np.random.default_rng(10).normal(size=(rays.shape[0], 3)).astype(np.float32)
    gs = torch.zeros(tree.n_leaves, device="cuda")
    gk = torch.zeros((tree.n_leaves, B, 3), device="cuda")
    po.po_render_backward(tree, r, torch.from_numpy(g).cuda(), gs, gk, gamma=gamma)
    rs, rk = om.backward(ot, rays.astype(np.float32).astype(np.float64), g.astype(np.float64), gamma=gamma)
    for a, b, tag in ((gs.cpu().numpy(), rs, "sigma"), (gk.cpu().numpy(), rk, "sg coefficients")):
        a, b = a.ravel().astype(np.float64), b.ravel()
        assert np.linalg.norm(a - b) <= 1e-3 * np.linalg.norm(b), tag
    # back to SH: identical to a fresh SH tree
    tree.set_sg_basis(None)
    sh_out = po.po_render_rays(tree, r, gamma=gamma)
    assert torch.equal(sh_out, po.po_render_rays(po.tree_from_gen(t), r, gamma=gamma))
    with pytest.raises(po.PoError):
        tree.set_sg_basis(np.zeros((B, 3), np.float32), lam)


def test_sg_tree_scratch_growth_keeps_lobes(env):
    """Scratch growth must not touch the tree's other device buffers (round-1 advisor finding:
    po_backward_plan's growth freed the deterministic scratch and the SG lobes): an SG tree runs
    the deterministic backward, then po_backward_plan on a larger batch (its scratch grows), then
    renders and backpropagates again -- identical to a fresh SG tree -- and is destroyed."""
    po, om, torch = env
    t = gen.scene_random(79, depth=5, sh_degree=2, sigma_scale=3.0)
    axes, lam = _sg_lobes(9, 11)
    tree = po.tree_from_gen(t)
    tree.set_sg_basis(axes, lam)
    fresh = po.tree_from_gen(t)
    fresh.set_sg_basis(axes, lam)
    rays = torch.from_numpy(gen.random_rays(80, 2000, inside_frac=0.1)).cuda()
    n = rays.shape[0]
    g = torch.randn((n, 3), device="cuda")
    aux = torch.empty((n, 4), dtype=torch.float64, device="cuda")
    seg = po.Segments(n, 64)
    po.po_render_rays(tree, rays, aux=aux, gamma=0.0, segments=seg)
    gs = torch.zeros(tree.n_leaves, device="cuda")
    gk = torch.zeros((tree.n_leaves, 9, 3), device="cuda")
    po.po_render_backward_deterministic(tree, rays, g, gs, gk, aux, seg, gamma=0.0)
    for m in (100, 50000):   # the plan scratch grows on the second call
        span = torch.zeros((m, 2), dtype=torch.int32, device="cuda")
        po.po_backward_plan(tree, span, 4)
    torch.cuda.synchronize()
    assert torch.equal(po.po_render_rays(tree, rays, gamma=0.01), po.po_render_rays(fresh, rays, gamma=0.01))
    gs2, gk2 = torch.zeros_like(gs), torch.zeros_like(gk)
    po.po_render_backward_deterministic(tree, rays, g, gs2, gk2, aux, seg, gamma=0.0)
    assert torch.equal(gs, gs2) and torch.equal(gk, gk2)
    tree.destroy()
    fresh.destroy()

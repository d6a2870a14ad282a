"""NEXT f2 on the GPU: the optimisation loop (epochs, validation-PSNR early stopping with
restore of the best epoch), leaf snapshot / restore, and the fp16 export."""
import numpy as np
import pytest

import gen
from conftest import rng

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


def _setup(po, c0_tree, n_train=6, seed=80, noise=(0.5, 0.3)):
    cams = np.concatenate([gen.orbit_camera(3.0, 30.0 * i, 20.0, 64, 64, 70.0) for i in range(n_train + 2)])
    gt = po.tree_from_gen(c0_tree)
    rays = po.po_camera_rays(po.cams_tensor(cams), 64, 64).reshape(-1, 6)
    target = po.po_render_rays(gt, rays, gamma=0.0)
    nt = n_train * 64 * 64
    g = rng(seed)
    sig = (c0_tree.sigma + g.normal(0.0, noise[0], c0_tree.sigma.shape)).astype(np.float32)
    sh = (c0_tree.sh + g.normal(0.0, noise[1], c0_tree.sh.shape)).astype(np.float32)
    tree = po.po_tree_create(c0_tree.child, sig, sh, c0_tree.depth, 1, c0_tree.bbox_min, c0_tree.edge)
    return tree, rays[:nt].contiguous(), target[:nt].contiguous(), rays[nt:].contiguous(), target[nt:].contiguous()


def test_trainer_improves_validation_psnr(env, c0_tree):
    po, torch = env
    from paper_2103_14024_b200.train import Trainer
    tree, r, t, vr, vt = _setup(po, c0_tree)
    tr = Trainer(tree, r, t, vr, vt, lr=2e4, batch_rays=4096, max_epochs=6, patience=2, reduction="mean")
    hist = tr.fit()
    assert max(hist) > hist[0] + 0.5, hist          # better than the perturbed tree
    assert len(tr.train_loss) >= 2 and tr.train_loss[-1] < tr.train_loss[0]
    # the tree ends at the best validation epoch
    assert abs(tr.validation_psnr() - max(hist)) < 1e-3


def test_early_stopping_restores_best(env, c0_tree):
    """A learning rate that overshoots: validation PSNR falls, training stops after `patience`
    epochs and the tree is restored to the best (here: the initial) leaves."""
    po, torch = env
    from paper_2103_14024_b200.train import Trainer
    tree, r, t, vr, vt = _setup(po, c0_tree, noise=(0.05, 0.02))
    s0, k0 = tree.read_leaves()
    tr = Trainer(tree, r, t, vr, vt, lr=1e7, batch_rays=4096, max_epochs=10, patience=1, reduction="mean")
    hist = tr.fit()
    assert len(hist) <= 1 + 10 and hist[1] < hist[0], hist
    assert len(hist) == 2                            # stopped after one non-improving epoch
    s1, k1 = tree.read_leaves()
    np.testing.assert_array_equal(s1, s0)
    np.testing.assert_array_equal(k1, k0)


def test_write_leaves_roundtrip_and_validation(env, c0_tree):
    po, torch = env
    tree = po.tree_from_gen(c0_tree)
    s, k = tree.read_leaves()
    g = rng(3)
    s2 = (s + g.normal(size=s.shape)).astype(np.float32)
    k2 = (k + g.normal(size=k.shape)).astype(np.float32)
    tree.write_leaves(s2, k2)
    a, b = tree.read_leaves()
    np.testing.assert_array_equal(a, s2)
    np.testing.assert_array_equal(b, k2)
    bad = s2.copy()
    bad[7] = np.nan
    with pytest.raises(po.PoError):
        tree.write_leaves(bad, k2)
    np.testing.assert_array_equal(tree.read_leaves()[0], s2)   # nothing written on error


def test_export_f16(env):
    """fp16 export: coefficients rounded to nearest-even, sigma~ kept in fp32 (reading
    Q20), same structure (identical traces), render within the fp16 budget of reading Q29."""
    po, torch = env
    t = gen.scene_random(91, depth=6, sh_degree=3, sigma_scale=3.0)
    tree = po.tree_from_gen(t)
    q = po.po_tree_convert(tree, po.PO_F16)
    s, k = q.read_leaves()
    np.testing.assert_array_equal(s, t.sigma)
    np.testing.assert_array_equal(k, t.sh.astype(np.float16).astype(np.float32))
    rays = torch.from_numpy(gen.random_rays(92, 3000)).cuda()
    ia, ca, _ = po.po_trace(tree, rays, max_leaves=32, gamma=0.0)
    ib, cb, _ = po.po_trace(q, rays, max_leaves=32, gamma=0.0)
    assert torch.equal(ia, ib) and torch.equal(ca, cb)
    a = po.po_render_rays(tree, rays).cpu().numpy()
    b = po.po_render_rays(q, rays).cpu().numpy()
    assert np.abs(a - b).max() <= 2e-3
    from paper_2103_14024_b200.train import export_f16
    q2 = export_f16(tree)
    assert q2.desc.payload == po.PO_F16

"""a9 / SURVEY 8(e) at N = 2 with the real kernels: two gloo ranks sharing the one GPU each take
half of a ray batch and run OctreeOptimizer.step (forward, Eq. 3, pass 2, SUM of the ranks'
gradients, SGD) in every gradient-sync mode: bucketed allreduce, the 4-chunk pass 2 overlapped
with the allreduce (stored segments and re-traversal), reduce-scatter + shard SGD + all-gather.

Eq. (3) is a sum over rays, so the summed gradient of the two halves IS the
full-batch gradient: every mode's updated tree must match the oracle's full-batch gradient step
(bars of reading Q26) and the single-rank full-batch step, both ranks must hold the same tree,
and the deterministic allreduce and reduce-scatter paths must agree bit for bit after 3 steps
(tools/rs_vs_ar.py folded in)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import gen
from conftest import rng

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED, DEPTH, DEG = 60, 5, 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grad_ok(a, b, tag):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    rel = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)
    assert rel <= 1e-3, f"{tag}: rel L2 {rel:.3e}"
    tol = 1e-3 * np.abs(b) + 1e-6 * np.abs(b).max()
    bad = np.abs(a - b) > tol
    assert not bad.any(), f"{tag}: {bad.sum()} components outside tolerance, worst {np.abs(a - b).max():.3e}"


@pytest.fixture(scope="module")
def runs(oracle_mod, tmp_path_factory):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import __graft_entry__ as g
    g.build()
    om = oracle_mod
    t = gen.scene_random(SEED, depth=DEPTH, sh_degree=DEG, sigma_scale=3.0)
    rays = gen.random_rays(SEED + 1, 6000, inside_frac=0.1)
    ot = om.OracleTree(t)
    r64 = rays.astype(np.float64)
    ok = om.tie_flags(ot, r64, gamma=1e-30) == 0
    rays = np.ascontiguousarray(rays[ok])
    target = rng(SEED + 2).random((rays.shape[0], 3)).astype(np.float32)
    d = tmp_path_factory.mktemp("multirank")
    np.savez(d / "case.npz", seed=SEED, depth=DEPTH, deg=DEG, rays=rays, target=target)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "tests", "helpers", "multirank_worker.py"), "--dir", str(d)]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    return t, rays, target, d


def _load(d, name, rank):
    z = np.load(d / f"{name}_r{rank}.npz")
    return z["sigma"], z["sh"], float(z["loss"])


@pytest.mark.parametrize("mode", ["allreduce", "chunks4", "chunks4_retraverse", "reduce_scatter"])
def test_two_ranks_equal_full_batch_oracle_step(runs, oracle_mod, mode):
    import torch
    import paper_2103_14024_b200 as po
    from paper_2103_14024_b200.optim import OctreeOptimizer
    t, rays, target, d = runs
    om = oracle_mod
    s0, k0, loss0 = _load(d, mode, 0)
    s1, k1, loss1 = _load(d, mode, 1)
    # both replicas hold the same tree after the step (the update used the same summed gradient)
    np.testing.assert_array_equal(s0, s1)
    np.testing.assert_array_equal(k0, k1)
    # the oracle's full-batch Eq. (3) gradient and loss
    ot = om.OracleTree(t)
    r64 = rays.astype(np.float64)
    ref = om.render(ot, r64, gamma=0.0)
    diff = ref["rgb"] - target.astype(np.float64)
    assert abs(loss0 - (diff ** 2).sum()) <= 1e-5 * (diff ** 2).sum()
    gs, gk = om.backward(ot, r64, 2.0 * diff, gamma=0.0)
    lr = 1.0
    _grad_ok((t.sigma.astype(np.float64) - s0) / lr, gs, f"{mode} sigma")
    _grad_ok((t.sh.astype(np.float64) - k0) / lr, gk, f"{mode} sh")
    # the single-rank full-batch step on the same GPU
    tree = po.tree_from_gen(t)
    OctreeOptimizer(tree, lr=lr, gamma=0.0, max_seg=16).step(torch.from_numpy(rays).cuda(),
                                                            torch.from_numpy(target).cuda())
    s, k = tree.read_leaves()
    _grad_ok((t.sigma.astype(np.float64) - s0), (t.sigma.astype(np.float64) - s), f"{mode} vs 1 rank sigma")
    _grad_ok((t.sh.astype(np.float64) - k0), (t.sh.astype(np.float64) - k), f"{mode} vs 1 rank sh")


def test_deterministic_reduce_scatter_equals_allreduce_bitwise(runs):
    """Order-fixed pass 2 on both ranks: the reduce-scatter SGD and the allreduce SGD leave
    bit-identical trees after 3 steps, on both ranks, and the tree moved."""
    t, _, _, d = runs
    ref = _load(d, "det_allreduce", 0)
    for rank in (0, 1):
        for name in ("det_allreduce", "det_reduce_scatter"):
            s, k, _ = _load(d, name, rank)
            np.testing.assert_array_equal(s, ref[0])
            np.testing.assert_array_equal(k, ref[1])
    assert not np.array_equal(ref[1], t.sh)

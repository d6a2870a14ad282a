"""Small driver for compute-sanitizer: every kernel of libplenoct on config c0 sizes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2103_14024_b200 as po  # noqa: E402
from paper_2103_14024_b200.optim import OctreeOptimizer  # noqa: E402

t = gen.scene_c0()
tree = po.tree_from_gen(t)
cam, W, H = gen.config_camera("c0")
ct = po.cams_tensor(cam)
img = po.po_render(tree, ct, W, H)
for _ in range(3):   # cost-ordered hand-out: order rewrite by the last CTA, split blocks (nb = 16)
    po.po_render(tree, ct, W, H)
po.po_render(tree, ct, 40, 24)   # stream order table re-initialised for another size
rays = po.po_camera_rays(ct, W, H).reshape(-1, 6)
out = po.po_render_rays(tree, rays)
aux = torch.empty((rays.shape[0], 4), dtype=torch.float64, device="cuda")
po.po_render_rays(tree, rays, aux=aux, gamma=0.0)
gs = torch.zeros(tree.n_leaves, device="cuda")
gk = torch.zeros((tree.n_leaves, 4, 3), device="cuda")
g = torch.randn((rays.shape[0], 3), device="cuda")
po.po_render_backward(tree, rays, g, gs, gk, gamma=0.0)
po.po_render_backward(tree, rays, g, gs, gk, aux=aux, gamma=0.0)
po.po_trace(tree, rays, max_leaves=16)
po.po_trace(tree, rays, max_leaves=16, classic=True)
po.po_render_stats(tree, ct, W, H)
opt = OctreeOptimizer(tree, lr=1.0)
opt.step(rays, out)
# stored segments (overflow path too), chunk plan + chunked replay, sparse SGD with zeroing
for ms in (64, 2):
    o2 = OctreeOptimizer(tree, lr=1.0, max_seg=ms, chunks=3)
    o2.step(rays, out)
    o3 = OctreeOptimizer(tree, lr=1.0, max_seg=ms, chunks=1)
    o3.step(rays, out)
o4 = OctreeOptimizer(tree, lr=1.0, max_seg=2, deterministic=True)   # segmented reduction + overflow
o4.step(rays, out)
# NEXT rows: depth / alpha, max alpha, SH-25, SG basis, fp16 export, leaf write
po.po_render_depth(tree, rays)
po.po_leaf_max_alpha(tree, rays)
t4 = po.tree_from_gen(gen.scene_random(5, depth=5, sh_degree=4))
po.po_render(t4, ct, W, H)
ax = np.random.default_rng(0).normal(size=(25, 3)).astype(np.float32)
t4.set_sg_basis(ax, np.full(25, 4.0, np.float32))
r4 = po.po_render_rays(t4, rays)
g4s = torch.zeros(t4.n_leaves, device="cuda")
g4k = torch.zeros((t4.n_leaves, 25, 3), device="cuda")
po.po_render_backward(t4, rays, g, g4s, g4k, gamma=0.0)
q4 = po.po_tree_convert(t4, po.PO_F16)
po.po_render(q4, ct, W, H)
s_, k_ = tree.read_leaves()
tree.write_leaves(s_, k_)
tq = po.tree_from_gen(gen.scene_random(3, depth=6, sh_degree=3), payload=po.PO_F16)
po.po_render(tq, ct, W, H)
po.po_render_host(tree, cam, W, H)
torch.cuda.synchronize()
print("sanitize driver done")

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
po.po_render_stats(tree, ct, W, H)
opt = OctreeOptimizer(tree, lr=1.0)
opt.step(rays, out)
tq = po.tree_from_gen(gen.scene_random(3, depth=6, sh_degree=3), payload=po.PO_F16)
po.po_render(tq, ct, W, H)
po.po_render_host(tree, cam, W, H)
torch.cuda.synchronize()
print("sanitize driver done")

"""How often do rays that run together in pass 2 write the same leaf?  c4 batch (1 M rays,
8x4-tile sampling, ordered by first-entered leaf as bench.py builds it), pass 1 with stored
segments, then for groups of G consecutive rays (G = 1 warp-per-ray CTA of 8, 32, ...): segments
per unique (group, leaf) pair -- the reduction factor an aggregation inside such a group gives."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2103_14024_b200 as po  # noqa: E402

W = H = 800
t_gt = gen.scene_c1()
gt = po.tree_from_gen(t_gt)
g = np.random.Generator(np.random.Philox(key=1))
sig = (t_gt.sigma + g.normal(0.0, 0.1 * 768.0, t_gt.sigma.shape)).astype(np.float32)
sh = (t_gt.sh + g.normal(0.0, 0.1, t_gt.sh.shape)).astype(np.float32)
tree = po.po_tree_create(t_gt.child, sig, sh, t_gt.depth, 3, t_gt.bbox_min, t_gt.edge)
cams = gen.fibonacci_hemisphere(100, 4.0, W, H, 1111.111)
rg = np.random.Generator(np.random.Philox(key=2 + 5))
n_rays = 1 << 20
tx_n, ty_n = W // 8, H // 4
tiles = rg.choice(100 * tx_n * ty_n, size=n_rays // 32, replace=False)
tiles.sort()
tv, tr_ = tiles // (tx_n * ty_n), tiles % (tx_n * ty_n)
x0, y0 = (tr_ % tx_n) * 8, (tr_ // tx_n) * 4
lane = np.arange(32)
pix = (y0[:, None] + lane[None] // 8) * W + x0[:, None] + lane[None] % 8
pick = (tv[:, None] * (W * H) + pix).reshape(-1)
rays = torch.from_numpy(gen.camera_rays_f32(cams, W, H, pick // (W * H), pick % (W * H))).cuda()
mode = sys.argv[1] if len(sys.argv) > 1 else "leaf"
if mode == "leaf":
    ids, _, _ = po.po_trace(gt, rays, max_leaves=1, gamma=0.0, with_nodes=False)
    key = ids[:, 0].to(torch.int64)
    key = torch.where(key < 0, torch.full_like(key, 1 << 40), key)
    rays = rays[torch.argsort(key, stable=True)].contiguous()
n = rays.shape[0]
seg = po.Segments(n, 256)
aux = torch.empty((n, 4), dtype=torch.float64, device="cuda")
po.po_render_rays(tree, rays, aux=aux, gamma=0.0, segments=seg)
cnt = seg.count.cpu().numpy()
rec = seg.records[:, :, 0].contiguous().view(torch.int32).cpu().numpy()   # [max_seg][n] leaf ids
valid = np.arange(256)[:, None] < np.minimum(cnt, 256)[None, :]
ray_id = np.broadcast_to(np.arange(n)[None, :], rec.shape)[valid].astype(np.int64)
leaf = rec[valid].astype(np.int64)
print(f"order {mode}: rays {n}, segments {leaf.size}, unique leaves {np.unique(leaf).size} of {tree.n_leaves}")
for G in (1, 8, 32, 128, 1024, 8192):
    u = np.unique((ray_id // G) << 32 | leaf).size
    print(f"group of {G:5d} consecutive rays: {leaf.size / u:.2f} segments per (group, leaf)")

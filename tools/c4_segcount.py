"""Distribution of sigma~>0 segments per ray in the c4 batch (sizes po_segments.max_seg)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2103_14024_b200 as po  # noqa: E402

t_gt = gen.scene_c1()
g = np.random.Generator(np.random.Philox(key=1))
sig = (t_gt.sigma + g.normal(0.0, 0.1 * 768.0, t_gt.sigma.shape)).astype(np.float32)
sh = (t_gt.sh + g.normal(0.0, 0.1, t_gt.sh.shape)).astype(np.float32)
tree = po.po_tree_create(t_gt.child, sig, sh, t_gt.depth, 3, t_gt.bbox_min, t_gt.edge)
cams = gen.fibonacci_hemisphere(100, 4.0, 800, 800, 1111.111)
rg = np.random.Generator(np.random.Philox(key=2))
pick = rg.choice(100 * 800 * 800, size=1 << 20, replace=False)
rays = torch.from_numpy(gen.camera_rays_f32(cams, 800, 800, pick // (800 * 800), pick % (800 * 800))).cuda()
n = rays.shape[0]
seg = po.Segments(n, 1024)
aux = torch.empty((n, 4), dtype=torch.float64, device="cuda")
po.po_render_rays(tree, rays, aux=aux, gamma=0.0, segments=seg)
c = seg.count.cpu().numpy()
hit = c[c > 0]
print("rays", n, "with sigma>0 segments", hit.size, "total segments", int(c.sum()))
print("per hitting ray: mean %.1f p50 %d p90 %d p99 %d p99.9 %d max %d" % (
    hit.mean(), *np.percentile(hit, [50, 90, 99, 99.9]).astype(int), hit.max()))
for m in (64, 96, 128, 192, 256, 384):
    print(f"max_seg {m}: overflow rays {(c > m).sum()} ({100 * (c > m).mean():.3f} %)")

"""Diagnostics for c1 parity: po_render vs po_render_rays(po_camera_rays) and the worst pixels."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import oracle  # noqa: E402
import paper_2103_14024_b200 as po  # noqa: E402

t = gen.scene_c1()
tree = po.tree_from_gen(t)
cam, W, H = gen.config_camera("c1")
cams = po.cams_tensor(cam)
img = po.po_render(tree, cams, W, H, gamma=0.01).reshape(-1, 3)
grays = po.po_camera_rays(cams, W, H).reshape(-1, 6)
img2 = po.po_render_rays(tree, grays, gamma=0.01)
print("po_render vs po_render_rays(po_camera_rays): max diff", (img - img2).abs().max().item())
img = img.cpu().numpy()
g32 = grays.cpu().numpy()
rays = oracle.camera_rays(cam, W, H)
ot = oracle.OracleTree(t)
pick = np.random.Generator(np.random.Philox(key=17)).choice(W * H, 4096, replace=False)
ref = oracle.render(ot, rays[pick], gamma=0.01, max_leaves=64)
ref32 = oracle.render(ot, g32[pick].astype(np.float64), gamma=0.01, max_leaves=64)
err = np.abs(img[pick] - ref["rgb"]).max(1)
err32 = np.abs(img[pick] - ref32["rgb"]).max(1)
print("max err vs oracle(double camera rays)", err.max(), " vs oracle(GPU fp32 rays)", err32.max())
for i in np.argsort(-err32)[:3]:
    p = pick[i]
    print(f"pixel {p}: err32 {err32[i]:.3e} gpu {img[p]} oracle32 {ref32['rgb'][i]} nproc {ref32['n_proc'][i]}")
    r = torch.from_numpy(g32[p:p + 1]).cuda()
    ids, cnt, nodes = po.po_trace(tree, r, max_leaves=64, gamma=0.01)
    print("  gpu ids", ids[0][:cnt[0].item()].tolist(), "nodes", nodes[0].item())
    lf, a, b, tnf = oracle.trace_ray(ot, g32[p].astype(np.float64))
    print("  oracle segs", [(int(x), float(y), float(z)) for x, y, z in zip(lf[:10], a[:10], b[:10])], tnf)
    print("  ray", g32[p].tolist())

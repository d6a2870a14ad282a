"""Renders c1 views 0..V-1 (and a c0 view) with the current PO_RENDER_OPT into OUT.npz, or
compares two such files: python tools/ab_images.py render OUT | compare A B"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if sys.argv[1] == "compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in a.files:
        x, y = a[k], b[k]
        d = np.abs(x.astype(np.float64) - y)
        px = (d.reshape(-1, 3).max(axis=1) > 0).sum()
        print(f"{k}: pixels differing {px} of {d.size // 3}, max |diff| {d.max():.3g}")
    sys.exit(0)
import torch  # noqa: E402
import gen  # noqa: E402
import paper_2103_14024_b200 as po  # noqa: E402
t = gen.scene_c1()
tree = po.tree_from_gen(t)
cams = po.cams_tensor(np.concatenate([gen.config_camera("c1", v)[0] for v in range(8)]))
imgs = {f"c1_v{v}": po.po_render(tree, cams[v:v + 1], 800, 800).cpu().numpy() for v in range(8)}
c0 = gen.scene_c0()
t0 = po.tree_from_gen(c0)
cam0 = po.cams_tensor(gen.config_camera("c0", 0)[0])
imgs["c0"] = po.po_render(t0, cam0, 64, 64).cpu().numpy()
np.savez(sys.argv[2], **imgs)

"""Per-box-step cycles of the slowest c1 warp tile (po_ray_step_timing): the tile's 32 rays in
one warp vs its longest ray alone.  Groups steps by (descent loads, box level, previous box a
shaded leaf) to show where the critical path's cycles go."""
import os
import sys
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2103_14024_b200 as po  # noqa: E402

t = gen.scene_c1()
tree = po.tree_from_gen(t)
cams = po.cams_tensor(np.concatenate([gen.config_camera("c1", v)[0] for v in range(8)]))
rays_all = po.po_camera_rays(cams[6:7], 800, 800).reshape(800, 800, 6)
x0, y0 = int(os.environ.get("TX", 552)), int(os.environ.get("TY", 436))   # slowest tile of view 6 (diag_tail)
tile = rays_all[y0:y0 + 4, x0:x0 + 8].reshape(-1, 6).contiguous()
_, cnt, nodes = po.po_trace(tree, tile, max_leaves=0, gamma=0.01)
k = int(torch.argmax(nodes).item())


def run(r, label, reps=5):
    for _ in range(2):
        po.po_ray_step_timing(tree, r)
    torch.cuda.synchronize()
    recs = []
    for _ in range(reps):
        rec, steps = po.po_ray_step_timing(tree, r)
        torch.cuda.synchronize()
        recs.append((rec.cpu().numpy().view(np.uint32), steps.cpu().numpy()))
    rec, steps = recs[-1]
    lane = k if r.shape[0] > 1 else 0
    ns = int(steps[lane])
    cyc = rec[lane, :ns, 0].astype(np.int64)
    info = rec[lane, :ns, 1]
    loads, shift, leafp = info >> 8, (info >> 1) & 15, info & 1
    print(f"== {label}: longest ray (lane {k}) {ns} box steps, {cyc.sum()} cycles "
          f"({cyc.sum() / 1.965e3:.1f} us at 1965 MHz), {loads.sum()} child-entry loads, {leafp.sum()} shaded leaves")
    groups = defaultdict(list)
    for c, l, s, lp in zip(cyc, loads, shift, leafp):
        groups[(int(min(l, 4)), int(min(s, 3)), int(lp))].append(int(c))
    print("  (loads, box shift, prev leaf): steps, mean cycles, median, total share")
    for key in sorted(groups):
        v = np.array(groups[key])
        print(f"  {key}: {len(v):4d} {v.mean():8.0f} {np.median(v):8.0f} {v.sum() / cyc.sum():6.1%}")
    if r.shape[0] > 1:
        tot = np.array([rec[j, :min(int(steps[j]), rec.shape[1]), 0].astype(np.int64).sum() for j in range(r.shape[0])])
        print(f"  per-lane total cycles: max {tot.max()} mean {tot.mean():.0f}; steps max {steps.max()} mean "
              f"{steps.mean():.1f}")


run(tile, "32-lane tile")
run(tile[k:k + 1].contiguous(), "longest ray alone")
run(tile[k:k + 1].repeat(32, 1).contiguous(), "longest ray x32")

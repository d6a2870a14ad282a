"""Phase structure of one single-view frame (c1 or c3) under the production schedule (cost-ordered
hand-out after 5 warm-up views on the stream): tiles in flight per 10 us, per-SM last tile end,
the slowest tiles.  Diagnostics build (PO_NVCC_EXTRA=-DPO_DIAG).  Usage: timeline_view.py c1|c3"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2103_14024_b200 as po  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c1"
if wl == "c3":
    tree = po.tree_from_gen(gen.scene_c3(), payload=po.PO_F16)
    W, H = 1920, 1080
else:
    tree = po.tree_from_gen(gen.scene_c1())
    W, H = 800, 800
cams = po.cams_tensor(np.concatenate([gen.config_camera(wl, v)[0] for v in range(8)]))
fa = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
fb = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for i in range(6):
    po.po_render(tree, cams[i:i + 1], W, H)
fa.fill_(1.0)
fb.sum()
torch.cuda.synchronize()
_, tl = po.po_render_timeline(tree, cams[6:7], W, H)
torch.cuda.synchronize()
tl = tl.cpu().numpy().astype(np.int64)
ok = tl[:, 0] > 0
t0, t1, sm = tl[ok, 0], tl[ok, 1], tl[ok, 2] >> 32
split = (tl[ok, 3] >> 32) != 0
base = t0.min()
t0 = (t0 - base) / 1e3
t1 = (t1 - base) / 1e3
dur = t1 - t0
span = t1.max()
print(f"{wl}: {ok.sum()} warp tiles ({split.sum()} of split blocks), span {span:.1f} us")
print("tile duration us: p50 %.1f p90 %.1f p99 %.1f max %.1f" % tuple(np.percentile(dur, [50, 90, 99, 100])))
last_end = np.array([t1[sm == s].max() for s in np.unique(sm)])
print("per-SM last tile end us: min %.1f p10 %.1f p50 %.1f max %.1f" % (
    last_end.min(), np.percentile(last_end, 10), np.percentile(last_end, 50), last_end.max()))
bins = np.arange(0, span + 10, 10)
print("tiles in flight per 10 us:", [int(((t0 <= b) & (t1 > b)).sum()) for b in bins])
pos = np.flatnonzero(ok) // 8
top = np.argsort(-t1)[:12]
print("last 12 tiles to end (hand-out pos, split, start, dur):",
      [(int(pos[j]), bool(split[j]), round(float(t0[j]), 1), round(float(dur[j]), 1)) for j in top])

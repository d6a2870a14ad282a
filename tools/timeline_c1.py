"""Scheduling analysis of one c1 frame: per-tile start/end times from po_render_timeline.
Needs a diagnostics build: PO_NVCC_EXTRA=-DPO_DIAG (po_render_timeline is refused otherwise)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2103_14024_b200 as po  # noqa: E402

t = gen.scene_c1()
tree = po.tree_from_gen(t)
V = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cams = po.cams_tensor(np.concatenate([gen.config_camera("c1", v)[0] for v in range(20 * V)]))
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for i in range(5):
    po.po_render(tree, cams[i * V:(i + 1) * V], 800, 800)
flush.zero_()
torch.cuda.synchronize()
img, tl = po.po_render_timeline(tree, cams[6 * V:7 * V], 800, 800)
torch.cuda.synchronize()
tl = tl.cpu().numpy().astype(np.int64)
handed = (tl[:, 3] >> 32)
print(f"rays handed to helper warps: {int(handed.sum())} from {int((handed > 0).sum())} tiles")
t0, t1 = tl[:, 0], tl[:, 1]
sm = tl[:, 2] >> 32
ok = t0 > 0
t0, t1, sm = t0[ok], t1[ok], sm[ok]
base = t0.min()
t0 = (t0 - base) / 1e3
t1 = (t1 - base) / 1e3
span = t1.max()
dur = t1 - t0
print(f"V={V}: {ok.sum()} tiles, span {span:.1f} us (first start 0, last end {span:.1f})")
print("tile duration us: p50 %.1f p90 %.1f p99 %.1f max %.1f mean %.1f" % (
    np.percentile(dur, 50), np.percentile(dur, 90), np.percentile(dur, 99), dur.max(), dur.mean()))
last_end = np.array([t1[sm == s].max() for s in np.unique(sm)])
print("per-SM last tile end us: min %.1f p10 %.1f p50 %.1f max %.1f (SMs %d)" % (
    last_end.min(), np.percentile(last_end, 10), np.percentile(last_end, 50), last_end.max(), len(last_end)))
first_start = np.array([t0[sm == s].min() for s in np.unique(sm)])
print("per-SM first tile start us: max %.1f" % first_start.max())
# warps active over time (tiles in flight), 10 us bins
bins = np.arange(0, span + 10, 10)
inflight = [((t0 <= b) & (t1 > b)).sum() for b in bins]
print("tiles in flight per 10 us:", inflight)
order = np.argsort(t0)
late = order[int(0.95 * len(order)):]
print("last 5%% of tiles started after %.1f us, their mean duration %.1f us" % (t0[late].min(), dur[late].mean()))
early = np.flatnonzero(sm == sm[np.argmin(t0)])
early = early[np.argsort(t0[early])][:24]
sub_all = np.flatnonzero(ok) % 8
print("tiles of one SM in start order (t0, t1, sub):",
      [(round(float(t0[j]), 1), round(float(t1[j]), 1), int(sub_all[j])) for j in early])
# the slowest tiles: where are they and what do their rays do
if V == 1:
    rec = tl[ok]
    blk = rec[:, 2] & 0xFFFFFFFF
    idx = np.flatnonzero(ok)
    sub = idx % 8
    rays = po.po_camera_rays(cams[6:7], 800, 800).reshape(800, 800, 6)
    bx_n = 50
    for j in np.argsort(-dur)[:6]:
        b, s = int(blk[j]), int(sub[j])
        x0, y0 = (b % bx_n) * 16 + (s & 1) * 8, (b // bx_n) * 16 + (s >> 1) * 4
        r = rays[y0:y0 + 4, x0:x0 + 8].reshape(-1, 6).contiguous()
        _, cnt, nodes = po.po_trace(tree, r, max_leaves=0, gamma=0.01)
        print(f"tile at x={x0} y={y0}: start {t0[j]:.1f} dur {dur[j]:.1f} us; leaves/ray max {cnt.max().item()} "
              f"mean {cnt.float().mean().item():.1f}; nodes/ray max {nodes.max().item()} mean {nodes.float().mean().item():.1f}")

"""Is the c1 single-frame drain a per-ray critical path or contention?  Times the slowest warp
tiles of one frame (from po_render_timeline) rendered ALONE through po_render_rays (one warp),
next to their in-frame duration, plus the per-ray box / node / leaf counts of those tiles."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2103_14024_b200 as po  # noqa: E402

t = gen.scene_c1()
tree = po.tree_from_gen(t)
cams = po.cams_tensor(np.concatenate([gen.config_camera("c1", v)[0] for v in range(8)]))
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for i in range(5):
    po.po_render(tree, cams[i:i + 1], 800, 800)
flush.zero_()
torch.cuda.synchronize()
img, tl = po.po_render_timeline(tree, cams[6:7], 800, 800)
torch.cuda.synchronize()
tl = tl.cpu().numpy().astype(np.int64)
ok = tl[:, 0] > 0
idx = np.flatnonzero(ok)
rec = tl[ok]
t0 = (rec[:, 0] - rec[:, 0].min()) / 1e3
t1 = (rec[:, 1] - rec[:, 0].min()) / 1e3
dur = t1 - t0
blk = rec[:, 2] & 0xFFFFFFFF
sub = idx % 8
print(f"frame span {t1.max():.1f} us, {len(dur)} tiles")
pos = idx // 8   # hand-out position of the tile's block (centre-out order)
for q in (50, 90, 99, 99.9):
    print(f"  tile duration p{q}: {np.percentile(dur, q):.1f} us")
for thr in (100, 120, 140, 160):
    sel = t1 > thr
    print(f"  tiles ending after {thr} us: {int(sel.sum())}, their hand-out positions p50 {np.median(pos[sel]) if sel.any() else -1:.0f} max {pos[sel].max() if sel.any() else -1}")
top30 = np.argsort(-t1)[:30]
print("  last 30 tiles to finish (hand-out pos, start, dur):", [(int(pos[j]), round(float(t0[j]), 1), round(float(dur[j]), 1)) for j in top30])
topd = np.argsort(-dur)[:30]
print("  30 longest tiles (hand-out pos, start, dur):", [(int(pos[j]), round(float(t0[j]), 1), round(float(dur[j]), 1)) for j in topd])
rays_all = po.po_camera_rays(cams[6:7], 800, 800).reshape(800, 800, 6)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
top = np.argsort(-dur)[:12]
tiles = []
for j in top:
    b, s = int(blk[j]), int(sub[j])
    x0, y0 = (b % 50) * 16 + (s & 1) * 8, (b // 50) * 16 + (s >> 1) * 4
    r = rays_all[y0:y0 + 4, x0:x0 + 8].reshape(-1, 6).contiguous()
    tiles.append(r)
    out = torch.empty(32, 3, device="cuda")
    for _ in range(3):
        po.po_render_rays(tree, r, out=out)
    ts = []
    for _ in range(10):
        ev0.record()
        po.po_render_rays(tree, r, out=out)
        ev1.record()
        torch.cuda.synchronize()
        ts.append(ev0.elapsed_time(ev1) * 1e3)
    _, cnt, nodes = po.po_trace(tree, r, max_leaves=0, gamma=0.01)
    print(f"tile x={x0:3d} y={y0:3d} start {t0[j]:6.1f} in-frame {dur[j]:6.1f} us | alone {np.median(ts):6.1f} us | "
          f"leaves max {cnt.max().item():3d} mean {cnt.float().mean().item():5.1f} | nodes max {nodes.max().item():3d} "
          f"mean {nodes.float().mean().item():5.1f}")
# all 12 slowest tiles together, one warp each (concurrency without the rest of the frame)
r = torch.cat(tiles)
out = torch.empty(r.shape[0], 3, device="cuda")
ts = []
for _ in range(10):
    ev0.record()
    po.po_render_rays(tree, r, out=out)
    ev1.record()
    torch.cuda.synchronize()
    ts.append(ev0.elapsed_time(ev1) * 1e3)
print(f"12 slowest tiles in one launch: {np.median(ts):.1f} us")
# empty-launch overhead reference
r1 = tiles[0][:1].contiguous()
o1 = torch.empty(1, 3, device="cuda")
ts = []
for _ in range(10):
    ev0.record()
    po.po_render_rays(tree, r1, out=o1)
    ev1.record()
    torch.cuda.synchronize()
    ts.append(ev0.elapsed_time(ev1) * 1e3)
print(f"one ray of the slowest tile alone: {np.median(ts):.1f} us")
# the slowest ray replicated on all 32 lanes (identical paths, no divergence), and the slowest
# tile's rays reduced to 8 / 16 lanes (the rest masked by n)
def alone(r):
    o = torch.empty(r.shape[0], 3, device="cuda")
    ts = []
    for _ in range(10):
        ev0.record()
        po.po_render_rays(tree, r, out=o)
        ev1.record()
        torch.cuda.synchronize()
        ts.append(ev0.elapsed_time(ev1) * 1e3)
    return np.median(ts)
_, cnt0, nodes0 = po.po_trace(tree, tiles[0], max_leaves=0, gamma=0.01)
k = int(torch.argmax(nodes0).item())
print(f"slowest ray x32 (identical lanes): {alone(tiles[0][k:k + 1].repeat(32, 1).contiguous()):.1f} us")
for m in (1, 2, 4, 8, 16):
    print(f"slowest tile, first {m} lanes: {alone(tiles[0][:m].contiguous()):.1f} us")
for j in range(4):   # each of the 4 slowest tiles as two 8x2 halves (16 lanes each)
    print(f"tile {j}: 32 lanes {alone(tiles[j]):.1f} us, rows 0-1 {alone(tiles[j][:16].contiguous()):.1f} us, "
          f"rows 2-3 {alone(tiles[j][16:].contiguous()):.1f} us")

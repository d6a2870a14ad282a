"""Upper bound of a cost-ordered block hand-out for the c1 single frame (diagnostics build, run
with PO_RENDER_ORDER=centre so po_set_block_order decides the order).
For views v = 6..9: the per-block cost is measured with po_render_timeline (centre-out order),
then view v is timed (L2 flushed, CUDA events, median of 15) under
  centre-out | its own costs, costliest block first | the previous view's costs (temporal
  coherence of an orbit) | the previous view's costs dilated by one block."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2103_14024_b200 as po  # noqa: E402

WL = os.environ.get("WL", "c1")
if WL == "c3":
    W, H = 1920, 1080
    tree = po.tree_from_gen(gen.scene_c3(), payload=po.PO_F16)
else:
    W = H = 800
    tree = po.tree_from_gen(gen.scene_c1())
BX, BY = (W + 15) // 16, (H + 15) // 16
cams = po.cams_tensor(np.concatenate([gen.config_camera(WL, v)[0] for v in range(12)]))
flush_a = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
flush_b = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
centre = None


def flush():
    flush_a.fill_(1.0)
    flush_b.sum()


def cost_of(v):
    po.po_set_block_order(tree, W, H, centre)
    flush()
    _, tl = po.po_render_timeline(tree, cams[v:v + 1], W, H)
    torch.cuda.synchronize()
    tl = tl.cpu().numpy().astype(np.int64)
    dur = (tl[:, 1] - tl[:, 0]) / 1e3
    blk = tl[:, 2] & 0xFFFFFFFF
    c_max = np.zeros(BX * BY)
    c_sum = np.zeros(BX * BY)
    np.maximum.at(c_max, blk, dur)
    np.add.at(c_sum, blk, dur)
    return c_max, c_sum


def timed(v, order, n=15):
    po.po_set_block_order(tree, W, H, order)
    out = torch.empty((1, H, W, 3), device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(n):
        flush()
        e0.record()
        po.po_render(tree, cams[v:v + 1], W, H, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


# the library's centre-out order (distance of the block centre from the image centre, stable)
ids = np.arange(BX * BY)
dx = (ids % BX) * 16 + 8 - W / 2
dy = (ids // BX) * 16 + 8 - H / 2
centre = np.argsort(dx * dx + dy * dy, kind="stable").astype(np.uint32)
for _ in range(3):
    timed(0, centre, 3)


def by_cost(c):
    return np.argsort(-c, kind="stable").astype(np.uint32)


def dilate(c):
    g = c.reshape(BY, BX)
    p = np.pad(g, 1)
    m = np.max([p[1 + a:1 + a + BY, 1 + b:1 + b + BX] for a in (-1, 0, 1) for b in (-1, 0, 1)], axis=0)
    return m.ravel()


for v in (range(6, 10) if __name__ == "__main__" else ()):
    cm, cs = cost_of(v)
    pm, ps = cost_of(v - 1)
    r = {"centre": timed(v, centre), "own_max": timed(v, by_cost(cm)), "own_sum": timed(v, by_cost(cs)),
         "prev_max": timed(v, by_cost(pm)), "prev_max_dilated": timed(v, by_cost(dilate(pm))),
         "centre2": timed(v, centre)}
    print(f"view {v}: " + "  ".join(f"{k} {x:.1f}" for k, x in r.items()), flush=True)

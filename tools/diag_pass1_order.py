"""Does the order in which c4 pass 1 claims its 8x4 tiles matter?  One c4 batch (1 M rays, the
bench's tile sampling), pass 1 (po_render_rays with aux + stored segments, gamma 0) timed with
CUDA events (median of 7, L2 flushed) with the tiles in: tileleaf order (the bench), random
order, costliest tile first (per-tile max of the rays' leaf counts), cheapest first."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2103_14024_b200 as po  # noqa: E402

W = H = 800
t = gen.scene_c1()
tree = po.tree_from_gen(t)
cams = gen.fibonacci_hemisphere(100, 4.0, W, H, 1111.111)
rg = np.random.Generator(np.random.Philox(key=2))
tx_n, ty_n = W // 8, H // 4
n = 1 << 20
tiles = np.sort(rg.choice(100 * tx_n * ty_n, size=n // 32, replace=False))
tv, tr_ = tiles // (tx_n * ty_n), tiles % (tx_n * ty_n)
x0, y0 = (tr_ % tx_n) * 8, (tr_ // tx_n) * 4
lane = np.arange(32)
pix = (y0[:, None] + lane[None] // 8) * W + x0[:, None] + lane[None] % 8
pick = (tv[:, None] * (W * H) + pix).reshape(-1)
rays = torch.from_numpy(gen.camera_rays_f32(cams, W, H, pick // (W * H), pick % (W * H))).cuda()
ids, cnt, _ = po.po_trace(tree, rays, max_leaves=1, gamma=0.0, with_nodes=False)
key = ids[:, 0].to(torch.int64)
key = torch.where(key < 0, torch.full_like(key, 1 << 40), key).view(-1, 32).min(dim=1).values
tcost = cnt.view(-1, 32).max(dim=1).values
orders = {"tileleaf": torch.argsort(key, stable=True),
          "random": torch.from_numpy(np.random.default_rng(1).permutation(n // 32)).cuda(),
          "costliest_first": torch.argsort(-tcost, stable=True),
          "cheapest_first": torch.argsort(tcost, stable=True)}
out = torch.empty((n, 3), device="cuda")
aux = torch.empty((n, 4), dtype=torch.float64, device="cuda")
seg = po.Segments(n, 256)
fa = torch.empty(64 << 20, device="cuda")
fb = torch.empty(64 << 20, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
print(f"leaf visits per ray: mean {cnt.float().mean().item():.1f}, per-tile max: mean {tcost.float().mean().item():.1f} max {tcost.max().item()}")
for rnd in range(2):
    for name, o in orders.items():
        r = rays.view(-1, 32, 6)[o].reshape(-1, 6).contiguous()
        ts = []
        for _ in range(8):
            fa.fill_(1.0)
            fb.sum()
            e0.record()
            po.po_render_rays(tree, r, out=out, aux=aux, gamma=0.0, segments=seg)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        print(f"round {rnd} {name:16s} pass 1 {np.median(ts[1:]):7.1f} us", flush=True)

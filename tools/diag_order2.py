"""Which cost order is best for the c1 single frame (diagnostics build, PO_RENDER_ORDER=centre so
po_set_block_order decides): for views v = 6..11, block costs from view v-1 (po_render_timeline),
view v timed (L2 flushed, median of 15) under: the costliest block first; costliest and cheapest
alternating (each SM's first wave mixes one of each); the top 296 (one per CTA slot of the first
wave at 2 CTAs/SM) alternating with the cheapest, the rest costliest first."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from diag_order import BX, BY, H, W, by_cost, cams, centre, cost_of, timed  # noqa: E402


def zip_ends(o):
    z = []
    i, j = 0, len(o)
    while i < j:
        z.append(o[i]); i += 1
        if i < j:
            j -= 1; z.append(o[j])
    return np.array(z, dtype=np.uint32)


def top_mixed(o, k=296):
    top, rest = list(o[:k]), list(o[k:])
    cheap = rest[::-1][:k]
    mid = rest[:len(rest) - k]
    z = []
    for a, b in zip(top, cheap):
        z += [a, b]
    return np.array(z + mid, dtype=np.uint32)


tag = os.environ.get("PO_RENDER_MINB", "auto")
for v in range(6, 12):
    pm, _ = cost_of(v - 1)
    o = by_cost(pm)
    r = {"centre": timed(v, centre), "cost": timed(v, o), "zip": timed(v, zip_ends(o)), "top_mixed": timed(v, top_mixed(o))}
    print(f"minb {tag} view {v}: " + "  ".join(f"{k} {x:.1f}" for k, x in r.items()), flush=True)

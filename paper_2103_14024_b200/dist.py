"""Multi-GPU plumbing (torch.distributed): gradient buckets and the SUM allreduce of a9.

The optimisation step is data parallel over rays with the tree replicated on every rank;
Eq. (3) sums over rays, so the per-leaf gradients of the ranks are
SUMMED (reading Q23).  The gradient lives in one flat fp32 buffer

    flat = [ grad_sigma (n_leaves, padded to a multiple of 4) | grad_sh (n_leaves * 3B) ]

which is split into contiguous buckets.  Each bucket is allreduced asynchronously (NCCL over
NVLink/NVSwitch on a B200 box; gloo in the CPU tests) and the SGD update of a bucket's range
can start as soon as that bucket has arrived, overlapping the remaining transfers.
Rendering needs no collective: views are sharded across ranks.
"""
from __future__ import annotations

from typing import List, Tuple


def flat_layout(n_leaves: int, basis_dim: int) -> Tuple[int, int, int]:
    """(sigma_offset, sh_offset, total) in elements; sh rows stay 16-byte aligned."""
    pad = (n_leaves + 3) // 4 * 4
    return 0, pad, pad + n_leaves * 3 * basis_dim


def plan_buckets(total: int, bucket_elems: int, align: int = 1024) -> List[Tuple[int, int]]:
    """Contiguous [start, end) buckets covering [0, total) exactly once; starts aligned."""
    if total <= 0:
        return []
    bucket_elems = max(align, (bucket_elems + align - 1) // align * align)
    out = []
    s = 0
    while s < total:
        e = min(total, s + bucket_elems)
        out.append((s, e))
        s = e
    return out


def allreduce_buckets(flat, buckets, group=None):
    """Launch one async SUM allreduce per bucket; returns the work handles in bucket order."""
    import torch.distributed as dist
    works = []
    for s, e in buckets:
        works.append(dist.all_reduce(flat[s:e], op=dist.ReduceOp.SUM, group=group, async_op=True))
    return works


def flat_to_param_range(s: int, e: int, n_leaves: int, sh_offset: int) -> Tuple[int, int]:
    """Map a flat-buffer range to the parameter index space of po_tree_sgd_step_range
    ([0, n_leaves) = sigma~, then n_leaves + j = j-th SH element); padding is skipped."""
    def f(x):
        if x <= n_leaves:
            return x
        if x < sh_offset:
            return n_leaves
        return n_leaves + (x - sh_offset)
    return f(s), f(e)

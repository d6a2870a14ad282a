"""Multi-GPU plumbing (torch.distributed): gradient buckets and the SUM allreduce of a9.

The optimisation step is data parallel over rays with the tree replicated on every rank;
Eq. (3) sums over rays, so the per-leaf gradients of the ranks are
SUMMED (reading Q23).  The gradient lives in one flat fp32 buffer

    flat = [ grad_sigma (n_leaves, padded to a multiple of 4) | grad_sh (n_leaves * 3B) ]

which is split into contiguous buckets.  Each bucket is allreduced asynchronously (NCCL over
NVLink/NVSwitch on a B200 box; gloo in the CPU tests) and the SGD update of a bucket's range
can start as soon as that bucket has arrived, overlapping the remaining transfers.

`overlapped_chunks` goes further: pass 2 runs in K chunks planned by
po_backward_plan so that after chunk j the gradient of leaves [0, b_j) is final; that leaf
range (its sigma~ slice and its SH slice of `flat`) is allreduced while chunks j+1.. run.
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


def leaf_range_slices(a: int, b: int, n_leaves: int, basis_dim: int, sh_offset: int):
    """Leaves [a, b) -> ([flat ranges], [parameter ranges of po_tree_sgd_step_range])."""
    ne = 3 * basis_dim
    flat = [(a, b), (sh_offset + ne * a, sh_offset + ne * b)]
    param = [(a, b), (n_leaves + ne * a, n_leaves + ne * b)]
    return flat, param


def overlapped_chunks(flat, leaf_end, n_leaves: int, basis_dim: int, sh_offset: int, run_chunk, apply_final,
                      group=None, world_size: int = 1):
    """Drive pass 2 chunk by chunk with the allreduce of each newly final leaf range.

    run_chunk(j)        enqueue pass-2 chunk j (po_render_backward_chunk)
    apply_final(b, e)   update parameter range [b, e) once its gradient is summed (SGD)
    After chunk j every ray that writes leaves below leaf_end[j] has run (po_backward_plan),
    so the range [leaf_end[j-1], leaf_end[j]) is allreduced asynchronously while the later
    chunks are enqueued behind it; the updates follow in range order."""
    import torch.distributed as dist
    pending = []
    prev = 0
    for j, end in enumerate(leaf_end):
        run_chunk(j)
        fr, pr = leaf_range_slices(prev, int(end), n_leaves, basis_dim, sh_offset)
        works = []
        if world_size > 1:
            for s, e in fr:
                if e > s:
                    works.append(dist.all_reduce(flat[s:e], op=dist.ReduceOp.SUM, group=group, async_op=True))
        pending.append((works, pr))
        prev = int(end)
    for works, pr in pending:
        for w in works:
            w.wait()
        for b, e in pr:
            if e > b:
                apply_final(b, e)


def agree_bounds(bounds, n_leaves: int, group=None, world_size: int = 1):
    """Leaf bounds every rank will use: the mean of the ranks' calibrated bounds, floored.  The
    allreduce ranges of overlapped_chunks must be identical on all ranks (a collective of
    mismatched sizes fails), while each rank calibrates on its own rays.  A mean of
    non-decreasing sequences is non-decreasing and the last bound stays n_leaves."""
    b = [int(x) for x in bounds]
    if world_size <= 1:
        return b
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    t = torch.tensor(b, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    out = [int(v) for v in torch.floor(t / world_size).tolist()]
    out[-1] = int(n_leaves)
    for j in range(1, len(out)):
        out[j] = max(out[j], out[j - 1])
    return out


def shard_chunk(n_leaves: int, world_size: int, align: int = 4) -> int:
    """Leaves per rank for the reduce-scatter SGD: equal chunks, a multiple of `align` (keeps
    every shard's SH gradient rows 16-B aligned), covering n_leaves; chunk * world_size may run
    past n_leaves into the tree's zeroed spare leaves (po_tree_leaf_payload)."""
    c = -(-max(1, n_leaves) // max(1, world_size))
    return -(-c // align) * align


def reduce_scatter_sgd(flat_sigma, flat_sh, ne: int, n_leaves: int, chunk: int, rank: int, world_size: int, sgd_shard,
                       payload_sigma, payload_sh, group=None):
    """SGD fused into the gradient collective (NEXT f2): reduce-scatter gives rank r the summed
    gradient of leaves [r c, (r+1) c) only, the rank updates that shard (sgd_shard(gs, gk, b, e)
    with e clipped to n_leaves) -- 1/N of the update work -- and an in-place all-gather writes
    every rank's updated shard into every tree.  Same bytes on the wire as allreduce + SGD."""
    import torch
    import torch.distributed as dist
    dev = flat_sigma.device
    gs = torch.empty(chunk, dtype=flat_sigma.dtype, device=dev)
    gk = torch.empty(chunk * ne, dtype=flat_sh.dtype, device=dev)
    dist.reduce_scatter_tensor(gs, flat_sigma[:chunk * world_size], group=group)
    dist.reduce_scatter_tensor(gk, flat_sh[:chunk * world_size * ne], group=group)
    b = rank * chunk
    e = min(n_leaves, b + chunk)
    if e > b:
        sgd_shard(gs, gk, b, e)
    dist.all_gather_into_tensor(payload_sigma[:chunk * world_size], payload_sigma[b:b + chunk], group=group)
    dist.all_gather_into_tensor(payload_sh[:chunk * world_size], payload_sh[b:b + chunk], group=group)

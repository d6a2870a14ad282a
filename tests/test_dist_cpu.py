"""Multi-process (world_size 2, gloo, CPU) checks of the a9 plumbing: bucket plan, SUM
allreduce of the flat gradient buffer, and the flat -> parameter-range mapping used by
po_tree_sgd_step_range.  (The kernels themselves need a GPU; see tests/test_gpu_*.py.)"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_14024_b200.dist import (agree_bounds, allreduce_buckets, flat_layout, flat_to_param_range,
                                        leaf_range_slices, overlapped_chunks, plan_buckets)


def test_plan_covers_exactly_once():
    for total in (1, 1000, 4096, 123457):
        for be in (1, 1024, 5000, 1 << 20):
            b = plan_buckets(total, be)
            assert b[0][0] == 0 and b[-1][1] == total
            assert all(b[i][1] == b[i + 1][0] for i in range(len(b) - 1))
            assert all(e > s for s, e in b)
    assert plan_buckets(0, 10) == []


def test_flat_to_param_range_partition():
    for n, B in ((5, 16), (8, 4), (1001, 16), (3, 1)):
        _, off, total = flat_layout(n, B)
        assert off % 4 == 0 and off >= n
        for be in (1024, 7 * 1024):
            covered = []
            for s, e in plan_buckets(total, be):
                b, f = flat_to_param_range(s, e, n, off)
                covered.extend(range(b, f))
            assert covered == list(range(n * (1 + 3 * B)))


def _worker(rank, world, port, n, B, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, off, total = flat_layout(n, B)
    g = torch.Generator().manual_seed(100 + rank)
    flat = torch.randn(total, generator=g)
    mine = flat.clone()
    works = allreduce_buckets(flat, plan_buckets(total, 1024), None)
    for w in works:
        w.wait()
    q.put((rank, mine.numpy(), flat.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_allreduce_sum_world2():
    n, B = 3001, 16
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_worker, args=(r, 2, port, n, B, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    want = res[0][1].astype(np.float64) + res[1][1].astype(np.float64)
    for _, _, got in res:
        np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-6)


def emulate_plan(keys, n_leaves, K, bounds=None):
    """What po_backward_plan computes (include/plenoct.h), written out: stable sort of the rays
    by lowest leaf, chunk j = rays with key in [b_{j-1}, b_j), b_j = n_leaves (j+1) // K unless
    given; quantile j = the key at position n_hit (j+1) // K of the sorted rays that have one."""
    keys = np.minimum(np.asarray(keys, np.int64), n_leaves)
    perm = np.argsort(keys, kind="stable")
    leaf_end = list(bounds) if bounds is not None else [n_leaves * (j + 1) // K for j in range(K)]
    sk = keys[perm]
    ends = [int(np.searchsorted(sk, b, side="left")) for b in leaf_end]
    n_hit = int(np.searchsorted(sk, n_leaves, side="left"))
    quant = []
    for j in range(K):
        pos = n_hit * (j + 1) // K
        quant.append(n_leaves if (j == K - 1 or pos >= n_hit) else int(sk[pos]))
    return perm, ends, leaf_end, quant


def test_leaf_range_slices_tile_the_parameters():
    for n, B, K in ((10, 4, 3), (1001, 16, 8), (7, 1, 7)):
        _, off, _ = flat_layout(n, B)
        params = []
        prev = 0
        for j in range(K):
            e = n * (j + 1) // K
            _, pr = leaf_range_slices(prev, e, n, B, off)
            params.extend(range(*pr[0]))
            prev = e
        prev = 0
        for j in range(K):
            e = n * (j + 1) // K
            _, pr = leaf_range_slices(prev, e, n, B, off)
            params.extend(range(*pr[1]))
            prev = e
        assert params == list(range(n * (1 + 3 * B)))


def _rays_of_rank(rank, n_leaves, n_rays):
    """Synthetic 'rays': each writes a few leaves >= its first leaf (as a traversal does)."""
    g = np.random.default_rng(7 + rank)
    rays = []
    for _ in range(n_rays):
        if g.random() < 0.1:
            rays.append(np.zeros(0, np.int64))   # touches no sigma>0 leaf
            continue
        first = int(g.integers(0, n_leaves))
        rest = g.integers(first, min(n_leaves, first + 200), size=int(g.integers(0, 6)))
        rays.append(np.unique(np.concatenate([[first], rest])))
    return rays


def _chunk_worker(rank, world, port, n, B, K, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, off, total = flat_layout(n, B)
    rays = _rays_of_rank(rank, n, 400)
    keys = [int(r[0]) if len(r) else n for r in rays]
    perm, ends, leaf_end, _ = emulate_plan(keys, n, K)
    flat = torch.zeros(total, dtype=torch.float64)
    ne = 3 * B

    def run_chunk(j):
        for i in perm[(ends[j - 1] if j else 0):ends[j]]:
            for leaf in rays[i]:
                flat[leaf] += 1.0 + i
                flat[off + ne * leaf: off + ne * (leaf + 1)] += 0.5 * (i + 1)

    params = torch.zeros(n * (1 + ne), dtype=torch.float64)
    seen = []

    def apply_final(b, e):
        seen.append((b, e))
        for p in range(b, e):
            params[p] = flat[p] if p < n else flat[off + (p - n)]

    overlapped_chunks(flat, leaf_end, n, B, off, run_chunk, apply_final, group=None, world_size=world)
    q.put((rank, params.numpy(), seen))
    dist.barrier()
    dist.destroy_process_group()


def test_overlapped_chunks_world2_equals_full_sum():
    """Every gradient range is allreduced after the last chunk that writes it (the
    po_backward_plan invariant) and the updates tile the parameter space once."""
    n, B, K = 997, 4, 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_chunk_worker, args=(r, 2, port, n, B, K, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=180) for _ in range(2)]
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    ne = 3 * B
    want = np.zeros(n * (1 + ne))
    for rank in range(2):
        for i, r in enumerate(_rays_of_rank(rank, n, 400)):
            for leaf in r:
                want[leaf] += 1.0 + i
                want[n + ne * leaf: n + ne * (leaf + 1)] += 0.5 * (i + 1)
    for _, params, seen in res:
        np.testing.assert_allclose(params, want, rtol=0, atol=1e-9)
        cov = sorted(x for b, e in seen for x in range(b, e))
        assert cov == list(range(n * (1 + ne)))


def _bounds_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 1000
    local = [[100, 400, 401, 1000], [300, 350, 900, 1000]][rank]   # each rank's own quantiles
    q.put((rank, agree_bounds(local, n, None, world)))
    dist.barrier()
    dist.destroy_process_group()


def test_agree_bounds_world2_identical_and_monotone():
    """Ranks calibrate chunk bounds on their own rays; the allreduce ranges must match, so the
    bounds are agreed (mean, floored, monotone, last = n_leaves) before use."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_bounds_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1] == [200, 375, 650, 1000]

"""Multi-process (world_size 2, gloo, CPU) checks of the a9 plumbing: bucket plan, SUM
allreduce of the flat gradient buffer, and the flat -> parameter-range mapping used by
po_tree_sgd_step_range.  (The kernels themselves need a GPU; see tests/test_gpu_*.py.)"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_14024_b200.dist import allreduce_buckets, flat_layout, flat_to_param_range, plan_buckets


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

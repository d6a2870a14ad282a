"""Worker of tests/test_gpu_multirank.py: one rank of a 2-rank (gloo) job whose ranks share one
GPU.  Each rank takes its half of a ray batch and runs OctreeOptimizer.step in several
gradient-sync modes (a9 / f2); the resulting trees are saved for the test to compare against a
single-rank full-batch step and the oracle's summed Eq. (3) gradient."""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import paper_2103_14024_b200 as po  # noqa: E402
from paper_2103_14024_b200.optim import OctreeOptimizer  # noqa: E402

MODES = {   # name -> OctreeOptimizer kwargs, steps
    "allreduce": (dict(chunks=1, max_seg=16, fused_sgd=False), 1),
    "chunks4": (dict(chunks=4, max_seg=16), 1),
    "chunks4_retraverse": (dict(chunks=4, max_seg=0), 1),
    "reduce_scatter": (dict(reduce_scatter=True, max_seg=16), 1),
    "det_allreduce": (dict(chunks=1, deterministic=True, max_seg=64), 3),
    "det_reduce_scatter": (dict(reduce_scatter=True, deterministic=True, max_seg=64), 3),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", required=True)
    ap.add_argument("--lr", type=float, default=1.0)
    args = ap.parse_args()
    dist.init_process_group("gloo")
    rank, ws = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)   # every rank on the one GPU of the box
    d = np.load(os.path.join(args.dir, "case.npz"))
    t = gen.scene_random(int(d["seed"]), depth=int(d["depth"]), sh_degree=int(d["deg"]), sigma_scale=3.0)
    rays, target = d["rays"], d["target"]
    half = (rays.shape[0] + ws - 1) // ws
    mine = slice(rank * half, min(rays.shape[0], (rank + 1) * half))
    r = torch.from_numpy(np.ascontiguousarray(rays[mine])).cuda()
    tg = torch.from_numpy(np.ascontiguousarray(target[mine])).cuda()
    for name, (kw, steps) in MODES.items():
        tree = po.tree_from_gen(t)
        opt = OctreeOptimizer(tree, lr=args.lr, gamma=0.0, **kw)
        assert opt.world_size == ws
        losses = []
        for _ in range(steps):
            losses.append(opt.step(r, tg).item())
        torch.cuda.synchronize()
        tot = torch.tensor([losses[0]], dtype=torch.float64)
        dist.all_reduce(tot)
        s, k = tree.read_leaves()
        assert not opt.flat.any().item(), name   # every consumed gradient range was zeroed
        np.savez(os.path.join(args.dir, f"{name}_r{rank}.npz"), sigma=s, sh=k, loss=float(tot.item()))
        tree.destroy()
        dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

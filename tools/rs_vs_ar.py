"""2 ranks (torchrun, gloo, one GPU is enough): the reduce-scatter SGD and the allreduce SGD give
bit-identical trees after a few deterministic steps (run under torch.distributed.run)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2103_14024_b200 as po  # noqa: E402
from paper_2103_14024_b200.optim import OctreeOptimizer  # noqa: E402

dist.init_process_group("gloo")
rank, ws = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
t = gen.scene_c0()
cams = np.concatenate([gen.orbit_camera(3.0, 30.0 * i + 7 * rank, 20.0, 64, 64, 70.0) for i in range(3)])
gt = po.tree_from_gen(t)
rays = po.po_camera_rays(po.cams_tensor(cams), 64, 64).reshape(-1, 6)
target = po.po_render_rays(gt, rays, gamma=0.0)
g = np.random.default_rng(5)
sig = (t.sigma + g.normal(0.0, 0.5, t.sigma.shape)).astype(np.float32)
sh = (t.sh + g.normal(0.0, 0.3, t.sh.shape)).astype(np.float32)
leaves = {}
for mode in ("allreduce", "reduce_scatter"):
    tree = po.po_tree_create(t.child, sig, sh, t.depth, 1, t.bbox_min, t.edge)
    opt = OctreeOptimizer(tree, lr=0.5, gamma=0.0, chunks=1, deterministic=True,
                          reduce_scatter=(mode == "reduce_scatter"))
    for _ in range(3):
        opt.step(rays, target)
    torch.cuda.synchronize()
    leaves[mode] = tree.read_leaves()
same = all(np.array_equal(a, b) for a, b in zip(leaves["allreduce"], leaves["reduce_scatter"]))
moved = not np.array_equal(leaves["allreduce"][1], sh)
print(f"rank {rank}: reduce-scatter == allreduce bitwise: {same}; tree moved: {moved}", flush=True)
dist.destroy_process_group()
sys.exit(0 if (same and moved) else 1)

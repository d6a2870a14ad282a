"""Direct PlenOctree optimisation step (§4.3; App. B.3).

One step on a ray batch, all compute in libplenoct kernels (this module only orders calls
and owns buffers):

  1. po_render_rays   forward + double-precision totals (pass 1 of P:949-957) -> rgb, aux
  2. po_l2_loss_grad  Eq. (3): dL/dC = 2 (C^ - C), loss = sum ||C^ - C||^2
  3. po_render_backward  pass 2: per-leaf dL/dsigma~ and dL/dk scatter-added (+=)
  4. SUM allreduce of the flat gradient in buckets (NCCL, only when world_size > 1)
  5. po_tree_sgd_step_range per bucket as soon as that bucket has landed (P:492, P:973 SGD)

gamma defaults to 0: the paper applies early stopping "at test-time" (reading Q12).
"""
from __future__ import annotations

import torch

from . import (po_l2_loss_grad, po_render_backward, po_render_rays, po_tree_sgd_step_range)
from .dist import allreduce_buckets, flat_layout, flat_to_param_range, plan_buckets


class OctreeOptimizer:
    def __init__(self, tree, lr: float, gamma: float = 0.0, background=(1.0, 1.0, 1.0), group=None,
                 bucket_mb: float = 64.0, device=None):
        self.tree = tree
        self.lr = float(lr)
        self.gamma = float(gamma)
        self.background = tuple(background)
        self.group = group
        self.device = torch.device("cuda", tree.device) if device is None else torch.device(device)
        n, B = tree.n_leaves, tree.B
        _, self.sh_off, total = flat_layout(n, B)
        self.flat = torch.zeros(total, dtype=torch.float32, device=self.device)
        self.grad_sigma = self.flat[:n]
        self.grad_sh = self.flat[self.sh_off:].view(n, B, 3)
        self.buckets = plan_buckets(total, int(bucket_mb * (1 << 20)) // 4)
        self._bufs = {}
        self.loss = torch.zeros(1, dtype=torch.float64, device=self.device)

    @property
    def world_size(self) -> int:
        import torch.distributed as dist
        return dist.get_world_size(self.group) if dist.is_available() and dist.is_initialized() else 1

    def _buffers(self, n: int):
        if n not in self._bufs:
            self._bufs[n] = (torch.empty((n, 3), dtype=torch.float32, device=self.device),
                             torch.empty((n, 4), dtype=torch.float64, device=self.device),
                             torch.empty((n, 3), dtype=torch.float32, device=self.device))
        return self._bufs[n]

    def step(self, rays: torch.Tensor, target: torch.Tensor) -> torch.Tensor:
        """rays [n][6] f32, target [n][3] f32 on this rank's device; returns the local loss (device f64)."""
        n = rays.shape[0]
        rgb, aux, dL = self._buffers(n)
        po_render_rays(self.tree, rays, out=rgb, aux=aux, gamma=self.gamma, background=self.background)
        po_l2_loss_grad(rgb, target, dL_dC=dL, loss=self.loss)
        self.flat.zero_()
        po_render_backward(self.tree, rays, dL, self.grad_sigma, self.grad_sh, aux=aux, gamma=self.gamma,
                           background=self.background)
        nl = self.tree.n_leaves
        if self.world_size > 1:
            works = allreduce_buckets(self.flat, self.buckets, self.group)
            for (s, e), w in zip(self.buckets, works):
                w.wait()   # makes the current stream wait for this bucket only
                b, f = flat_to_param_range(s, e, nl, self.sh_off)
                po_tree_sgd_step_range(self.tree, self.grad_sigma, self.grad_sh, self.lr, b, f)
        else:
            po_tree_sgd_step_range(self.tree, self.grad_sigma, self.grad_sh, self.lr, 0, nl * (1 + 3 * self.tree.B))
        return self.loss

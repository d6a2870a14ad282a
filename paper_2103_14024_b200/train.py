"""NEXT f2: the PlenOctree optimisation loop (§4.3; App. "PlenOctree
Optimization Details" P:971-973) around OctreeOptimizer.step.

* epochs over the training rays in a fresh seeded order each epoch, SGD at a constant
  learning rate (1e7 on NeRF-synthetic, 1.5e6 on Tanks&Temples) for at most
  `max_epochs` (80 / 40);
* the learning rates of P:971 belong to a loss averaged over the batch (reading Q35), so
  `reduction="mean"` divides the step by the batch size; `"sum"` is Eq. (3) as written;
* after every epoch the validation PSNR (test-time rendering, gamma 0.01) is measured and
  training stops early once it has not improved for `patience` epochs, restoring the best
  tree ("early stopping ... by monitoring the PSNR on the validation set");
* optimisation runs in fp32; `export_f16` stores the result with fp16 coefficients.

Every numeric step runs in libplenoct kernels (po_render_rays, po_l2_loss_grad,
po_render_backward, po_tree_sgd_step_range); this module orders calls and keeps history.
"""
from __future__ import annotations

import math
from typing import List

import torch

from . import PO_F16, po_l2_loss_grad, po_render_rays, po_tree_convert
from .optim import OctreeOptimizer


def psnr_from_sse(sse: float, n_values: int) -> float:
    """PSNR of colours in [0, 1]: 10 log10(1 / MSE), MSE = SSE / n_values."""
    mse = sse / max(1, n_values)
    return math.inf if mse <= 0.0 else -10.0 * math.log10(mse)


def should_stop(history: List[float], patience: int) -> bool:
    """True once the best validation PSNR is `patience` or more epochs old."""
    if not history:
        return False
    best = max(range(len(history)), key=lambda i: history[i])
    return len(history) - 1 - best >= patience


class Trainer:
    def __init__(self, tree, rays, rgb, val_rays, val_rgb, lr: float, batch_rays: int = 1 << 20,
                 max_epochs: int = 80, patience: int = 1, reduction: str = "mean", gamma: float = 0.0,
                 val_gamma: float = 0.01, seed: int = 0, **opt_kw):
        if reduction not in ("mean", "sum"):
            raise ValueError("reduction must be 'mean' or 'sum'")
        self.tree = tree
        self.rays, self.rgb = rays, rgb
        self.val_rays, self.val_rgb = val_rays, val_rgb
        self.batch = int(batch_rays)
        self.max_epochs = int(max_epochs)
        self.patience = int(patience)
        self.val_gamma = float(val_gamma)
        self.reduction = reduction
        self.opt = OctreeOptimizer(tree, lr=lr, gamma=gamma, device=rays.device, **opt_kw)
        self.lr = float(lr)
        self.gen = torch.Generator(device=rays.device)
        self.gen.manual_seed(int(seed))
        self.history: List[float] = []
        self.train_loss: List[float] = []
        self._best = None
        self._sse = torch.zeros(1, dtype=torch.float64, device=rays.device)

    def validation_psnr(self) -> float:
        pred = po_render_rays(self.tree, self.val_rays, gamma=self.val_gamma)
        po_l2_loss_grad(pred, self.val_rgb, loss=self._sse)
        return psnr_from_sse(float(self._sse.item()), self.val_rgb.numel())

    def epoch(self) -> float:
        n = self.rays.shape[0]
        perm = torch.randperm(n, generator=self.gen, device=self.rays.device)
        total = torch.zeros(1, dtype=torch.float64, device=self.rays.device)
        for s in range(0, n, self.batch):
            idx = perm[s:s + self.batch]
            m = idx.shape[0]
            self.opt.lr = self.lr / m if self.reduction == "mean" else self.lr
            total += self.opt.step(self.rays[idx].contiguous(), self.rgb[idx].contiguous())
        loss = float(total.item())
        self.train_loss.append(loss)
        return loss

    def fit(self) -> List[float]:
        """Runs epochs until max_epochs or early stopping; the tree ends at the best epoch."""
        self.history = [self.validation_psnr()]
        self._best = self.tree.read_leaves()
        for _ in range(self.max_epochs):
            self.epoch()
            self.history.append(self.validation_psnr())
            if self.history[-1] >= max(self.history[:-1]):
                self._best = self.tree.read_leaves()
            if should_stop(self.history, self.patience):
                break
        if self.history[-1] < max(self.history):
            self.tree.write_leaves(*self._best)   # restore the best validation epoch
        return self.history


def export_f16(tree):
    """The trained fp32 tree stored with fp16 coefficients."""
    return po_tree_convert(tree, PO_F16)

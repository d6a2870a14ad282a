"""Direct PlenOctree optimisation step (§4.3; App. B.3).

One step on a ray batch, all compute in libplenoct kernels (this module only orders calls
and owns buffers):

  1. po_render_rays   forward + double-precision totals (pass 1 of P:949-957) -> rgb, aux,
                      and (max_seg > 0) every sigma~>0 segment's (leaf, delta, w, T, c) stored
  2. po_l2_loss_grad  Eq. (3): dL/dC = 2 (C^ - C), loss = sum ||C^ - C||^2
  3. po_render_backward  pass 2: per-leaf dL/dsigma~ and dL/dk scatter-added (+=), replaying the
                      stored segments (re-traversing only rays with more than max_seg of them)
  4. SUM allreduce of the flat gradient in buckets (NCCL, only when world_size > 1)
  5. po_tree_sgd_step_range per bucket as soon as that bucket has landed (P:492, P:973 SGD)

On one replica (world_size 1, stored segments, fp32 tree) steps 3-5 are one call,
po_render_backward_sgd: -lr * gradient goes straight into the tree (fused_sgd=False keeps the
separate gradient + SGD passes).

With chunks = K > 1 (K = 4 by default when world_size > 1), steps 3-5 overlap:
pass 1 also records each ray's leaf span, po_backward_plan orders the rays into K chunks,
and the gradient range a chunk finalises is allreduced while the next chunks run
(dist.overlapped_chunks).

gamma defaults to 0: the paper applies early stopping "at test-time" (reading Q12).
"""
from __future__ import annotations

import torch

from . import (PO_F32, Segments, po_backward_plan, po_l2_loss_grad, po_render_backward, po_render_backward_chunk,
               po_render_backward_deterministic, po_render_backward_sgd, po_render_rays,
               po_tree_sgd_step_range)
from .dist import (agree_bounds, allreduce_buckets, flat_layout, flat_to_param_range, overlapped_chunks, plan_buckets,
                   reduce_scatter_sgd, shard_chunk)


class OctreeOptimizer:
    def __init__(self, tree, lr: float, gamma: float = 0.0, background=(1.0, 1.0, 1.0), group=None,
                 bucket_mb: float = 64.0, device=None, chunks=None, max_seg: int = 256,
                 deterministic: bool = False, reduce_scatter: bool = False, fused_sgd: bool = True):
        self.tree = tree
        self.lr = float(lr)
        self.gamma = float(gamma)
        self.background = tuple(background)
        self.group = group
        self.device = torch.device("cuda", tree.device) if device is None else torch.device(device)
        n, B = tree.n_leaves, tree.B
        # reduce-scatter SGD (NEXT f2): equal leaf chunks per rank; the flat gradient is padded
        # to chunk * world_size leaves in both regions so the collectives split it evenly
        self.reduce_scatter = bool(reduce_scatter) and self.world_size > 1
        self.chunk = shard_chunk(n, self.world_size) if self.reduce_scatter else 0
        if self.reduce_scatter:
            self.sh_off = self.chunk * self.world_size
            total = self.sh_off + self.sh_off * 3 * B
        else:
            _, self.sh_off, total = flat_layout(n, B)
        self.flat = torch.zeros(total, dtype=torch.float32, device=self.device)
        self.grad_sigma = self.flat[:n]
        self.grad_sh = self.flat[self.sh_off:self.sh_off + n * 3 * B].view(n, B, 3)
        self.buckets = plan_buckets(total, int(bucket_mb * (1 << 20)) // 4)
        self._bufs = {}
        self.loss = torch.zeros(1, dtype=torch.float64, device=self.device)
        # pass-2 chunks overlapped with the allreduce; None = 4 when world_size > 1, else 1
        self.chunks = chunks
        self._side = None
        self.leaf_bounds = {}   # K -> host leaf bounds of po_backward_plan (calibrated on first use)
        # stored pass-1 segments per ray (po_segments, max_seg * n * 32 B); 0 = re-traverse in pass 2
        self.max_seg = int(max_seg)
        # order-fixed pass 2 (po_render_backward_deterministic): bit-reproducible gradients
        self.deterministic = bool(deterministic)
        # one replica: pass 2 writes -lr * gradient straight into the tree (po_render_backward_sgd)
        self.fused_sgd = bool(fused_sgd)
        if self.deterministic and self.max_seg <= 0:
            raise ValueError("the deterministic backward replays stored segments: max_seg must be > 0")

    @property
    def world_size(self) -> int:
        import torch.distributed as dist
        return dist.get_world_size(self.group) if dist.is_available() and dist.is_initialized() else 1

    def _buffers(self, n: int):
        if n not in self._bufs:
            self._bufs[n] = (torch.empty((n, 3), dtype=torch.float32, device=self.device),
                             torch.empty((n, 4), dtype=torch.float64, device=self.device),
                             torch.empty((n, 3), dtype=torch.float32, device=self.device),
                             torch.empty((n, 2), dtype=torch.int32, device=self.device),
                             torch.empty(n, dtype=torch.int32, device=self.device),
                             Segments(n, self.max_seg, self.device) if self.max_seg > 0 else None)
        return self._bufs[n]

    def n_chunks(self) -> int:
        if self.chunks is not None:
            return max(1, int(self.chunks))
        return 4 if self.world_size > 1 else 1

    def train_from_host(self, host_batches) -> torch.Tensor:
        """Steps over (rays [n][6], target [n][3][, group_order]) batches in PINNED host memory, one step each.

        Batch i+1's host->device copy runs on a side stream while step i computes (two device
        buffers, each refilled only after the step that read it), and every step's loss is
        copied device->host into a pinned tensor without blocking.  Returns that pinned float64
        [len(host_batches)] tensor (reused by the next call with as many batches); it is valid
        once the current stream has completed (e.g. after torch.cuda.synchronize()).  Every step's inputs still cross PCIe and every loss
        comes back: the copies overlap compute instead of preceding it."""
        k = len(host_batches)
        if k == 0:
            return torch.empty(0, dtype=torch.float64)
        n = host_batches[0][0].shape[0]
        # pipeline resources are allocated once per batch size (pinned and device allocations
        # synchronise the device, so they stay out of the steady state)
        key = ("pipe", n)
        if key not in self._bufs:
            self._bufs[key] = (torch.cuda.Stream(self.device),
                               [(torch.empty((n, 6), dtype=torch.float32, device=self.device),
                                 torch.empty((n, 3), dtype=torch.float32, device=self.device),
                                 torch.empty((n + 31) // 32, dtype=torch.int32, device=self.device)) for _ in range(2)],
                               [torch.cuda.Event() for _ in range(2)])
        ordered = len(host_batches[0]) > 2 and host_batches[0][2] is not None
        copy, bufs, ready = self._bufs[key]
        if ("losses", k) not in self._bufs:
            self._bufs[("losses", k)] = torch.empty(k, dtype=torch.float64, pin_memory=True)
        losses = self._bufs[("losses", k)]
        main = torch.cuda.current_stream(self.device)
        copy.wait_stream(main)   # the copies start after everything already queued on main
        free = [None, None]

        def prefetch(i):
            b = i % 2
            with torch.cuda.stream(copy):
                if free[b] is not None:
                    copy.wait_event(free[b])   # step i-2 has finished reading buffer b
                bufs[b][0].copy_(host_batches[i][0], non_blocking=True)
                bufs[b][1].copy_(host_batches[i][1], non_blocking=True)
                if ordered:
                    bufs[b][2].copy_(host_batches[i][2], non_blocking=True)
                ready[b].record(copy)

        prefetch(0)
        for i in range(k):
            if i + 1 < k:
                prefetch(i + 1)
            b = i % 2
            main.wait_event(ready[b])
            loss = self.step(bufs[b][0], bufs[b][1], bufs[b][2] if ordered else None)
            free[b] = torch.cuda.Event()
            free[b].record(main)
            losses[i].copy_(loss.view(()), non_blocking=True)
        return losses

    def step(self, rays: torch.Tensor, target: torch.Tensor, group_order=None) -> torch.Tensor:
        """rays [n][6] f32, target [n][3] f32 on this rank's device; returns the local loss (device f64).
        group_order: optional int32 [ceil(n/32)] order in which pass 1 claims the batch's 32-ray
        groups (costliest first removes pass 1's tail; scheduling only)."""
        n = rays.shape[0]
        rgb, aux, dL, span, perm, seg = self._buffers(n)
        K = self.n_chunks()
        po_render_rays(self.tree, rays, out=rgb, aux=aux, gamma=self.gamma, background=self.background,
                       leaf_span=span if K > 1 else None, segments=seg, group_order=group_order)
        po_l2_loss_grad(rgb, target, dL_dC=dL, loss=self.loss)
        # the gradient buffer is zero here: it starts zeroed and every SGD call below zeroes
        # what it consumed (PO_SGD_ZERO_GRAD), which replaces a 0.7 GB memset per step
        nl = self.tree.n_leaves
        if self.reduce_scatter:
            K = 1
        if K > 1 and self.deterministic:
            raise ValueError("deterministic pass 2 is not combined with the chunked overlap")
        if K > 1:
            key = ("plan", K)
            if key not in self._bufs:
                self._bufs[key] = (torch.empty(K, dtype=torch.int64, device=self.device),
                                   torch.empty(K, dtype=torch.int64, device=self.device))
            ends, quant = self._bufs[key]
            bounds = self.leaf_bounds.get(K)
            _, ends, leaf_end = po_backward_plan(self.tree, span, K, leaf_bounds=bounds, perm=perm, chunk_ray_end=ends,
                                                 key_quantiles=quant if bounds is None else None)
            if bounds is None:
                # first chunked step: one host sync to read this batch's ray quantiles; later
                # steps reuse them as leaf bounds (equal-work chunks; batches of one scene
                # have similar first-leaf distributions, and any bounds are correct)
                self.leaf_bounds[K] = agree_bounds(quant.cpu().tolist(), nl, self.group, self.world_size)
            # chunks alternate between two side streams so one chunk's tail (its slowest rays)
            # overlaps the next chunk; the current stream joins chunk j before the allreduce of
            # the range chunk j finalises is enqueued on it (gradient atomics commute, so
            # concurrent chunks are safe; only the allreduce needs chunks 0..j complete)
            main = torch.cuda.current_stream(self.device)
            if self._side is None:
                self._side = [torch.cuda.Stream(self.device) for _ in range(2)]
            ready = torch.cuda.Event()
            ready.record(main)
            for st in self._side:
                st.wait_event(ready)

            def run_chunk(j):
                st = self._side[j % 2]
                po_render_backward_chunk(self.tree, rays, perm, ends, j, dL, self.grad_sigma, self.grad_sh, aux=aux,
                                         gamma=self.gamma, background=self.background, stream=st, segments=seg)
                done = torch.cuda.Event()
                done.record(st)
                main.wait_event(done)

            def apply_final(b, e):
                po_tree_sgd_step_range(self.tree, self.grad_sigma, self.grad_sh, self.lr, b, e, zero_grad=True)

            overlapped_chunks(self.flat, leaf_end, nl, self.tree.B, self.sh_off, run_chunk, apply_final,
                              group=self.group, world_size=self.world_size)
            return self.loss
        if (self.fused_sgd and self.world_size == 1 and not self.deterministic and seg is not None
                and self.tree.desc.payload == PO_F32):
            po_render_backward_sgd(self.tree, rays, dL, self.lr, self.grad_sigma, self.grad_sh, aux, seg,
                                   gamma=self.gamma, background=self.background)
            return self.loss
        if self.deterministic:
            po_render_backward_deterministic(self.tree, rays, dL, self.grad_sigma, self.grad_sh, aux, seg,
                                             gamma=self.gamma, background=self.background)
        else:
            po_render_backward(self.tree, rays, dL, self.grad_sigma, self.grad_sh, aux=aux, gamma=self.gamma,
                               background=self.background, segments=seg)
        if self.reduce_scatter:
            ne = 3 * self.tree.B
            sig_view, sh_view = self.tree.payload_views()

            def sgd_shard(gs, gk, b, e):   # gradient index b sits at gs[0] / gk[0]
                po_tree_sgd_step_range(self.tree, gs.data_ptr() - 4 * b, gk.data_ptr() - 4 * b * ne, self.lr, b, e)
                po_tree_sgd_step_range(self.tree, gs.data_ptr() - 4 * b, gk.data_ptr() - 4 * b * ne, self.lr,
                                       nl + b * ne, nl + e * ne)

            reduce_scatter_sgd(self.flat[:self.sh_off], self.flat[self.sh_off:], ne, nl, self.chunk,
                               torch.distributed.get_rank(self.group), self.world_size, sgd_shard, sig_view, sh_view,
                               self.group)
            self.flat.zero_()   # the shard buffers were consumed; the flat gradient starts at 0 again
            return self.loss
        if self.world_size > 1:
            works = allreduce_buckets(self.flat, self.buckets, self.group)
            for (s, e), w in zip(self.buckets, works):
                w.wait()   # makes the current stream wait for this bucket only
                b, f = flat_to_param_range(s, e, nl, self.sh_off)
                po_tree_sgd_step_range(self.tree, self.grad_sigma, self.grad_sh, self.lr, b, f, zero_grad=True)
        else:
            po_tree_sgd_step_range(self.tree, self.grad_sigma, self.grad_sh, self.lr, 0, nl * (1 + 3 * self.tree.B),
                                   zero_grad=True)
        return self.loss

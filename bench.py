#!/usr/bin/env python
"""Benchmark of the PlenOctree render hot path (BASELINE.json metric: 800x800 FPS and
Mrays/s, SH-3 512^3 PlenOctree, 1/2/4/8 B200, % of HBM peak).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one 800x800 frame of config c1 (depth-9 sparse octree, SH-3, fp32 payload,
gamma = 0.01) through po_render, inputs resident in HBM.  Views walk the c1 orbit
(az = 37 + 1.8 i deg) so consecutive steps render different frames, and L2 is flushed
before every timed step (a 256 MiB write, then a 256 MiB read of another buffer so the
write's dirty lines leave L2 before the timed region: every frame starts on a cold, clean L2);
each step is timed with CUDA events on the launching stream and only the render is inside
the events.  For N > 1 (torchrun) every
rank renders its own views (weak scaling, tree replicated, no collective in the timed
region) and the time is the max over ranks.

`--impl reference` times the CPU oracle (oracle/, double precision, OpenMP) on a bounded
sample of the same workload on this host's cores: the reference arm of this tier.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W = H = 800
GAMMA = 0.01
METRIC = "800x800 FPS, SH-3 512^3 PlenOctree (c1)"
C2_VIEWS = 200
UNIT = "frames/s"
L2_FLUSH_BYTES = 256 << 20
L2_DESC = ("flushed before every timed step: a 256 MiB write, then a 256 MiB read of a second buffer so the "
           "write's dirty lines are written back before the timed region (the render starts on a cold, clean "
           "L2); only the render is inside the CUDA events")


class L2Flush:
    """Outside the timed region: overwrite a buffer twice the L2 size (evicts the previous
    frame's lines), then read another one (the flush's own dirty lines go back to HBM here, not
    inside the next timed render).  --flush write keeps the write alone (round-1 behaviour)."""

    def __init__(self, dev, mode="write+read"):
        import torch
        self.mode = mode
        self.w = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
        self.r = torch.zeros(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev) if mode == "write+read" else None
        self.acc = torch.zeros(1, dtype=torch.float32, device=dev)

    def __call__(self):
        import torch
        self.w.zero_()
        if self.r is not None:
            torch.sum(self.r, dim=0, keepdim=True, out=self.acc)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _ncu_traffic(wl: str = "c1"):
    """(dram bytes, L2 bytes, source) per k_render launch of workload wl from the committed
    ncu --set full summary (tools/ncu_summary.py)."""
    path = os.path.join(ROOT, "profiles", "ncu_render_summary.json" if wl == "c1" else f"ncu_render_summary_{wl}.json")
    try:
        with open(path) as f:
            s = json.load(f)
        lts = s.get("lts_bytes_per_launch")
        return float(s["dram_bytes_per_launch"]), (float(lts) if lts else None), s.get("source", path)
    except Exception:
        return None, None, None


def _l2_peak():
    """Measured L2 read bandwidth (tools/micro/l2bw.cu, profiles/l2_peak.json), GB/s."""
    try:
        with open(os.path.join(ROOT, "profiles", "l2_peak.json")) as f:
            return float(json.load(f)["l2_read_gbs"]), "measured (profiles/l2_peak.json, tools/micro/l2bw.cu)"
    except Exception:
        return None, None


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()
        time.sleep(0.3)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.th.join(timeout=2)
        import statistics
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _dist():
    """(world size, rank, CUDA device index).  PO_BENCH_DEVICE pins every rank to one device:
    with PO_BENCH_BACKEND=gloo that exercises the multi-rank path on a single-GPU box."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("PO_BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    return ws, rank, local


def _init_pg(dev_index: int):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(dev_index)
    backend = os.environ.get("PO_BENCH_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
    else:
        dist.init_process_group(backend)


ORDER_DESC = ("16x16 blocks handed out costliest first by the per-block cost the previous single-view render "
              "on the stream measured (temporal coherence of the orbit; the first render centre-out; images do "
              "not depend on the order; DESIGN.md 6.1 v13)")


def _workload_desc(tree_gen, wl="c1", ws=1):
    if wl == "c2":
        return {"workload": "c2: the c1 tree (depth-9, "
                            f"{tree_gen.n_leaves} leaves, SH-3 fp32), a 200-view 800x800 orbit per step, gamma 0.01",
                "views": "az = 1.8*i deg, el 30 deg, r 3.4, f 1111.1 px, i = 0..199; rank r renders views "
                         f"i = r (mod {ws}) in ONE launch",
                "l2": L2_DESC,
                "global_batch": "200 views per step (all ranks)"}
    if wl in ("c3", "c3sh25"):
        deg = "SH-25 (l = 4, P:587-588)" if wl == "c3sh25" else "SH-3"
        return {"workload": f"{wl}: Tanks&Temples-shaped bounded scene, depth-10 sparse octree (1024^3), "
                            f"{tree_gen.n_leaves} leaves / {tree_gen.n_nodes} nodes, {deg} fp16 payload (sigma fp32), "
                            "1920x1080, gamma 0.01",
                "views": "orbit r 2.6, el 15 deg, az = 20 + 1.8*i deg, f 1400 px; rank r renders views r, r+N, ...",
                "l2": L2_DESC,
                "block_order": ORDER_DESC,
                "global_batch": "1 frame per rank per step"}
    thick = " thick shell sdf/h in (-8, +1) (SURVEY 8(d) paper-scale variant, P:669 mean 1.93 GB)," if wl == "c1thick" else ""
    return {"workload": f"{wl}: NeRF-synthetic-shaped SDF object, depth-9 sparse octree (512^3),{thick} "
                        f"{tree_gen.n_leaves} leaves / {tree_gen.n_nodes} nodes, SH-3 fp32 payload, 800x800, gamma 0.01",
            "views": "c1 orbit, az = 37 + 1.8*i deg, el 30 deg, r 3.4, f 1111.1 px; rank r renders views r, r+N, ...",
            "l2": L2_DESC,
            "block_order": ORDER_DESC,
            "global_batch": "1 frame per rank per step"}


def run_ours(args):
    import numpy as np
    import torch
    import gen
    import paper_2103_14024_b200 as po

    wl = args.workload
    c3like = wl.startswith("c3")
    W, H = (1920, 1080) if c3like else (800, 800)
    payload = po.PO_F16 if c3like else po.PO_F32
    metric = {"c3": "1920x1080 FPS, SH-3 depth-10 fp16 PlenOctree (c3)",
              "c3sh25": "1920x1080 FPS, SH-25 depth-10 fp16 PlenOctree (c3 scene at the paper's T&T basis)",
              "c1thick": "800x800 FPS, SH-3 512^3 PlenOctree, thick shell (paper-scale tree)",
              "c2": "views/s, 200-view 800x800 orbit, SH-3 512^3 PlenOctree (c2)"}.get(wl, METRIC)
    unit = "views/s" if wl == "c2" else UNIT
    ws, rank, local = _dist()
    if ws > 1:
        _init_pg(local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    po.lib()
    t_gen = {"c3": lambda: gen.scene_c3(), "c3sh25": lambda: gen.scene_c3(sh_degree=4),
             "c1thick": lambda: gen.scene_c1(thick=True)}.get(wl, lambda: gen.scene_c1())()
    tree = po.tree_from_gen(t_gen, payload=payload, device=local)
    if wl == "c2":
        # every step renders the whole 200-view orbit: rank r takes views r, r+N, ... in one launch
        mine = list(range(rank, C2_VIEWS, ws))
        V = len(mine)
        cam_recs = np.concatenate([gen.config_camera("c2", v)[0] for v in mine])
        n_views = V
    else:
        V = max(1, args.views_per_launch)
        n_views = max(args.steps + args.warmup, 1) * ws * V
        cam_cfg = "c3" if c3like else ("c1" if wl == "c1thick" else wl)
        cam_recs = np.concatenate([gen.config_camera(cam_cfg, v)[0] for v in range(n_views)])
    cams = po.cams_tensor(cam_recs, dev)
    out = torch.empty((V, H, W, 3), dtype=torch.float32, device=dev)
    flush = L2Flush(dev, args.flush)
    stream = torch.cuda.current_stream(dev)

    tile_shard = args.shard == "tile" and wl in ("c1", "c3", "c1thick", "c3sh25")

    def view_of(step):   # first of the V consecutive views rank `rank` renders at `step`
        if wl == "c2":
            return 0
        if tile_shard:   # every rank renders its blocks of the SAME view
            return (step * V) % n_views
        return ((step * ws + rank) * V) % n_views

    def render_step(v):
        if not tile_shard:
            po.po_render(tree, cams[v:v + V], W, H, out=out, gamma=GAMMA)
            return
        # single-view latency mode: interleaved 16x16 blocks per rank, then a SUM
        # allreduce of the zero-initialised images assembles the frame on every rank
        out.zero_()
        po.po_render_shard(tree, cams[v:v + V], W, H, rank, ws, out=out, gamma=GAMMA)
        if ws > 1:
            torch.distributed.all_reduce(out, op=torch.distributed.ReduceOp.SUM)

    # algorithmic bytes per launch, SURVEY.md §8(d) ALG_RAY: every leaf visit moves one unpadded
    # leaf record (sigma~ 4 B + 3B coefficients), every internal node the ray's processed interval
    # meets one 32-B child sector, every pixel 12 B of output -- counts of the classic descent,
    # the implementation-independent definition (the cell-index kernel reads fewer node sectors)
    B = t_gen.basis_dim
    row_bytes = 3 * B * (2 if payload == po.PO_F16 else 4)
    rec_bytes = 4 + row_bytes
    stats = {"leaf_visits": 0, "sh_rows": 0, "nodes": 0, "hit_rays": 0, "boxes": 0, "leaf_level_boxes": 0,
             "warp_boxes": 0}
    stat_steps = range(args.warmup, args.warmup + (1 if wl == "c2" else args.steps))
    for s in stat_steps:
        v = view_of(s)
        st = po.po_render_stats(tree, cams[v:v + V], W, H, gamma=GAMMA)
        for k in stats:
            stats[k] += st[k] * (args.steps if wl == "c2" else 1)   # c2: every step renders the same orbit
    K = max(args.steps, 1)
    alg_bytes = (stats["leaf_visits"] * rec_bytes + stats["nodes"] * 32) / K + W * H * 12 * V
    if tile_shard:
        alg_bytes /= ws   # each rank renders 1/N of the blocks (interleaved: an even share)

    for s in range(args.warmup):
        flush()
        render_step(view_of(s))
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    l0 = po.launch_count()
    evs = []
    for s in range(args.warmup, args.warmup + args.steps):
        if args.l2 == "flush":
            flush()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        v = view_of(s) if args.l2 != "same" else view_of(args.warmup)
        e0.record(stream)
        render_step(v)
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    launches = po.launch_count() - l0
    clk = clocks.stop()
    t_ms = sum(a.elapsed_time(b) for a, b in evs)
    t_max = t_ms
    if ws > 1:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_max = float(tt.item())
    ms_per_step = t_max / K
    fps = (C2_VIEWS if wl == "c2" else (V if tile_shard else ws * V)) * K / (t_max / 1e3)
    kernel_ms = t_ms / K   # one kernel launch per step

    # e2e: the same frames through the host-buffer C-ABI entry point (H2D cameras, D2H image)
    pinned = torch.empty((V, H, W, 3), dtype=torch.float32, pin_memory=True).numpy()
    cams_pinned = torch.empty((n_views, 16), dtype=torch.float32, pin_memory=True).numpy()
    cams_pinned[:] = np.frombuffer(np.ascontiguousarray(cam_recs).tobytes(), dtype=np.float32).reshape(-1, 16)
    e2e_ms = 0.0
    e2e_steps = min(K, 3 if wl == "c2" else 50)
    for s in range(2):
        po.po_render_host(tree, cams_pinned[view_of(s):view_of(s) + V], W, H, out_host=pinned, gamma=GAMMA)
    if ws > 1:
        torch.distributed.barrier()
    cams_dev = torch.empty((V, 16), dtype=torch.float32, device=dev)
    pinned_t = torch.from_numpy(pinned)
    for s in range(args.warmup, args.warmup + e2e_steps):
        flush()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        v = view_of(s)
        e0.record(stream)
        if tile_shard:   # H2D cameras, this rank's blocks, allreduce, D2H of the assembled frame
            cams_dev.copy_(torch.from_numpy(cams_pinned[v:v + V]), non_blocking=True)
            out.zero_()
            po.po_render_shard(tree, cams_dev, W, H, rank, ws, out=out, gamma=GAMMA)
            if ws > 1:
                torch.distributed.all_reduce(out, op=torch.distributed.ReduceOp.SUM)
            pinned_t.copy_(out, non_blocking=True)
        else:
            po.po_render_host(tree, cams_pinned[v:v + V], W, H, out_host=pinned, gamma=GAMMA)
        e1.record(stream)
        e1.synchronize()
        e2e_ms += e0.elapsed_time(e1)
    if ws > 1:
        tt = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_fps = (C2_VIEWS if wl == "c2" else (V if tile_shard else ws * V)) * e2e_steps / (e2e_ms / 1e3)

    if rank == 0:
        peak, peak_src = _peaks()
        achieved = alg_bytes / (kernel_ms / 1e3) / 1e9
        traffic, lts, tsrc = (_ncu_traffic(wl) if (wl != "c2" and V == 1) or (wl == "c2" and ws == 1)
                              else (None, None, None))   # the captured launch shape only
        l2_peak, l2_src = _l2_peak()
        # SURVEY §8(d) graded fraction: max(DRAM bytes / t / HBM peak, L2 bytes / t / L2 peak), the
        # bytes from the committed ncu capture of this launch shape, t the live kernel time
        graded = None
        if traffic is not None:
            d_frac = traffic / (kernel_ms / 1e3) / 1e9 / peak
            l_frac = (lts / (kernel_ms / 1e3) / 1e9 / l2_peak) if (lts is not None and l2_peak) else None
            graded = {"frac": round(max(d_frac, l_frac or 0.0), 4), "dram_frac": round(d_frac, 4),
                      "l2_frac": None if l_frac is None else round(l_frac, 4), "l2_peak_gbs": l2_peak,
                      "l2_peak_source": l2_src, "l2_bytes_per_launch": lts,
                      "def": "max(ncu dram bytes / t / HBM peak, ncu lts__t_bytes / t / L2 peak), t = live kernel time"}
        line = {
            "metric": metric, "value": round(fps, 2), "unit": unit, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
            "scaling": "strong" if (wl == "c2" or tile_shard) else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (procedural SDF scene, seeded)",
            "config": _workload_desc(t_gen, wl, ws)
                      | {"parallelism": (f"tile-sharded x{ws} (interleaved 16x16 blocks of one view, SUM allreduce of "
                                         "the image), tree replicated") if tile_shard
                         else f"view-sharded x{ws}, tree replicated"}
                      | ({"global_batch": f"{V} frames per rank per step (one launch)"} if V > 1 and wl != "c2"
                         else {})
                      | ({"l2": f"NOT flushed ({args.l2}): analysis only"} if args.l2 != "flush" else {})
                      | ({"l2": "flushed before every timed step by a 256 MiB write (dirty lines left in L2)"}
                         if args.l2 == "flush" and args.flush == "write" else {}),
            "mrays_per_s": round(fps * W * H / 1e6, 1),
            "leaf_visits_per_frame": stats["leaf_visits"] / (K * V),
            "traversal_per_frame": {"boxes": stats["boxes"] / (K * V),
                                    "leaf_level_boxes": stats["leaf_level_boxes"] / (K * V),
                                    "internal_nodes_met": stats["nodes"] / (K * V),
                                    "hit_rays": stats["hit_rays"] / (K * V),
                                    "simt_step_efficiency": round(stats["boxes"] / max(1, 32 * stats["warp_boxes"]),
                                                                  4)},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": f"po::k_render<{t_gen.sh_degree},{int(payload == po.PO_F16)}>", "peak_source": peak_src,
                         "alg_bytes_per_launch": round(alg_bytes),
                         "alg_bytes_def": f"SURVEY 8(d) ALG_RAY: leaf visits*{rec_bytes} B record + internal nodes "
                                          "met (classic descent)*32 B + 12 B/pixel out",
                         "traffic_source": tsrc, "graded": graded},
            "e2e": {"value": round(e2e_fps, 2), "unit": unit, "h2d_bytes_per_step": 64 * V,
                    "d2h_bytes_per_step": W * H * 12 * V,
                    "entry": ("po_render_shard + image allreduce, cameras H2D / frame D2H" if tile_shard
                              else "po_render_host (host cameras -> host image)")},
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if not args.no_cpu_baseline and ws == 1 and wl == "c1":
            line["cpu_baseline"] = cpu_baseline(t_gen, seconds=args.cpu_seconds)
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def run_c4(args):
    """Config c4: direct-optimisation step (forward + Eq. 3 gradient + backward + SUM allreduce +
    SGD), 1,048,576 rays per GPU per step (8 M at 8 GPUs), gamma = 0 (reading Q12)."""
    import numpy as np
    import torch
    import gen
    import paper_2103_14024_b200 as po
    from paper_2103_14024_b200.optim import OctreeOptimizer

    ws, rank, local = _dist()
    group = None
    if ws > 1:
        _init_pg(local)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    t_gt = gen.scene_c1()
    gt = po.tree_from_gen(t_gt, device=local)
    g = np.random.Generator(np.random.Philox(key=1))
    sig = (t_gt.sigma + g.normal(0.0, 0.1 * 768.0, t_gt.sigma.shape)).astype(np.float32)
    sh = (t_gt.sh + g.normal(0.0, 0.1, t_gt.sh.shape)).astype(np.float32)
    tree = po.po_tree_create(t_gt.child, sig, sh, t_gt.depth, 3, t_gt.bbox_min, t_gt.edge, device=local)
    cams = gen.fibonacci_hemisphere(100, 4.0, W, H, 1111.111)
    n_rays = args.rays
    batches = []
    for s in range(args.warmup + args.steps):
        rg = np.random.Generator(np.random.Philox(key=2 + s * ws + rank))
        if args.ray_sampling == "tile":
            # sample 8x4-pixel tiles without replacement (each pixel still at most once per
            # batch); a tile's 32 rays are consecutive, i.e. one coherent warp
            tx_n, ty_n = W // 8, H // 4
            tiles = rg.choice(100 * tx_n * ty_n, size=n_rays // 32, replace=False)
            tiles.sort()
            tv, tr_ = tiles // (tx_n * ty_n), tiles % (tx_n * ty_n)
            x0, y0 = (tr_ % tx_n) * 8, (tr_ // tx_n) * 4
            lane = np.arange(32)
            pix = (y0[:, None] + lane[None] // 8) * W + x0[:, None] + lane[None] % 8
            pick = (tv[:, None] * (W * H) + pix).reshape(-1)
        else:
            pick = rg.choice(100 * W * H, size=n_rays, replace=False)
        if args.ray_sampling == "pixel" and not args.unsorted:
            # batch preparation: order the sampled rays by (view, Morton(x, y)) so a warp's 32
            # rays are spatially coherent (shared descent paths, fewer divergent branches)
            view, p = pick // (W * H), pick % (W * H)
            x, y = (p % W).astype(np.uint64), (p // W).astype(np.uint64)
            mx = gen.trees._part1by2(x) | (gen.trees._part1by2(y) << np.uint64(1))
            pick = pick[np.argsort((view.astype(np.uint64) << np.uint64(44)) | mx, kind="stable")]
        rays = torch.from_numpy(gen.camera_rays_f32(cams, W, H, pick // (W * H), pick % (W * H))).to(dev)
        if args.ray_order == "tileleaf" and args.ray_sampling == "tile":
            # keep each 8x4 tile's 32 rays together (warp coherence) and order the TILES by
            # the lowest first-entered leaf among their rays (inter-warp locality)
            ids, cnt, _ = po.po_trace(gt, rays, max_leaves=1, gamma=0.0, with_nodes=False)
            key = ids[:, 0].to(torch.int64)
            key = torch.where(key < 0, torch.full_like(key, 1 << 40), key).view(-1, 32).min(dim=1).values
            order = torch.argsort(key, stable=True)
            rays = rays.view(-1, 32, 6)[order].reshape(-1, 6).contiguous()
            cnt = cnt.view(-1, 32)[order].reshape(-1)
        if args.ray_order == "leaf":
            # batch preparation: order rays by the first leaf they enter.  The tree structure is
            # fixed during optimisation, so this key is a per-pixel constant; leaves are
            # numbered in Morton order, so rays that meet the same surface patch (from any
            # view) run together and share leaf rows / gradient rows in L1/L2.
            ids, _, _ = po.po_trace(gt, rays, max_leaves=1, gamma=0.0, with_nodes=False)
            key = ids[:, 0].to(torch.int64)
            key = torch.where(key < 0, torch.full_like(key, 1 << 40), key)
            rays = rays[torch.argsort(key, stable=True)].contiguous()
        tgt = po.po_render_rays(gt, rays, gamma=0.0)   # targets: renders of the unperturbed tree
        gorder = None
        if args.pass1_order == "costliest":
            # pass 1 claims the batch's 32-ray groups costliest first: at gamma 0 a ray's leaf
            # count is a constant of the fixed tree structure, known to the loader
            if args.ray_order != "tileleaf" or args.ray_sampling != "tile":
                _, cnt, _ = po.po_trace(gt, rays, max_leaves=1, gamma=0.0, with_nodes=False)
            n_g = (rays.shape[0] + 31) // 32
            cost = torch.zeros(n_g * 32, dtype=torch.int32, device=dev)
            cost[:rays.shape[0]] = cnt
            gorder = torch.argsort(-cost.view(n_g, 32).max(dim=1).values, stable=True).to(torch.int32)
        batches.append((rays, tgt, gorder))
    torch.cuda.synchronize()
    gt.destroy()
    opt = OctreeOptimizer(tree, lr=args.lr, gamma=0.0, device=dev, chunks=args.chunks, max_seg=args.max_seg,
                          deterministic=args.deterministic, reduce_scatter=args.reduce_scatter,
                          fused_sgd=not args.unfused_sgd)
    # algorithmic bytes of the dominant kernel (k_backward, pass 2 with aux) over the timed batches
    visits = nodes = 0
    for rays, _, _ in batches[args.warmup:]:
        _, cnt, nd = po.po_trace(tree, rays, max_leaves=0, gamma=0.0)
        visits += int(cnt.sum().item())
        nodes += int(nd.sum().item())
    for s in range(args.warmup):
        opt.step(*batches[s])
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    l0 = po.launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    losses = []
    for s in range(args.warmup, args.warmup + args.steps):
        losses.append(opt.step(*batches[s]).clone())
    e1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    launches = po.launch_count() - l0
    clk = clocks.stop()
    t_ms = e0.elapsed_time(e1)
    t_max = t_ms
    if ws > 1:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_max = float(tt.item())
    K = args.steps
    rays_per_s = ws * K * n_rays / (t_max / 1e3)

    # e2e: the same steps through the public API from pinned HOST batches: every step copies its
    # rays + targets host -> device inside the timed region and reads the loss back (D2H)
    e2e_steps = min(K, 10)
    host = [(b[0].cpu().pin_memory(), b[1].cpu().pin_memory(), None if b[2] is None else b[2].cpu().pin_memory())
            for b in batches[args.warmup:args.warmup + e2e_steps]]
    opt.train_from_host(host[:2])   # untimed: allocates the pipeline's buffers and side stream
    host_losses = opt.train_from_host(host)   # untimed warm-up of the full-length call
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    # OctreeOptimizer.train_from_host: each step's H2D copy overlaps the previous step on a side
    # stream, each step's loss comes back by an async D2H copy into pinned memory
    host_losses = opt.train_from_host(host)
    f1.record(stream)
    torch.cuda.synchronize()
    assert np.isfinite(host_losses.numpy()).all()
    e2e_ms = f0.elapsed_time(f1)
    if ws > 1:
        tt = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = ws * e2e_steps * n_rays / (e2e_ms / 1e3)
    if rank == 0:
        peak, peak_src = _peaks()
        alg = (visits * (4 + 192 + 196) + nodes * 32) / K + n_rays * (24 + 12 + 32)
        # per visited leaf 2 record reads + the 196-B gradient RMW (588 B), a node
        # sector per internal node for each of the two traversals, rays/colours/targets
        alg_survey = (visits * 588 + nodes * 64) / K + n_rays * (24 + 12 + 32)
        fused = (opt.fused_sgd and ws == 1 and not args.deterministic and args.max_seg > 0 and opt.n_chunks() == 1)
        line = {
            "metric": "direct octree optimisation rays/s (c4: forward+backward+allreduce+SGD)",
            "value": round(rays_per_s, 1), "unit": "rays/s", "n_gpus": ws, "steps": K, "warmup": args.warmup,
            "ms_per_step": round(t_max / K, 4), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (c1 tree perturbed; targets = renders of the unperturbed tree)",
            "config": {"workload": f"c4: {n_rays} rays per GPU per step from 100 Fibonacci-hemisphere 800x800 views, "
                                   "gamma 0, SGD lr %g" % args.lr, "parallelism": f"ray data-parallel x{ws}, "
                                   "tree replicated, bucketed NCCL SUM allreduce",
                       "ray_sampling": args.ray_sampling + ("" if args.ray_sampling == "tile" or not args.unsorted
                                                           else " (unsorted)"),
                       "ray_order": args.ray_order,
                       "pass1_claim_order": ("32-ray groups costliest first (per-group max leaf count at gamma 0, a "
                                             "per-pixel constant of the fixed structure, computed by the batch loader)"
                                             if args.pass1_order == "costliest" else "batch order"),
                       "pass2_chunks": opt.n_chunks(),
                       "pass2_reduction": "deterministic segmented" if args.deterministic else "atomic",
                       "gradient_sync": ("reduce-scatter + shard SGD + all-gather" if opt.reduce_scatter else
                                         ("allreduce overlapped with pass-2 chunks" if opt.n_chunks() > 1 else
                                          ("bucketed allreduce" if ws > 1 else "none (1 GPU)"))),
                       "pass2": (f"stored segments (max {args.max_seg}/ray, {args.max_seg * n_rays * 32 / 2**30:.1f} GiB)"
                                 if args.max_seg > 0 else "re-traversal"),
                       "update": ("SGD fused into pass 2 (po_render_backward_sgd: -lr*gradient added straight "
                                  "into the tree, no gradient buffer)" if fused else
                                  "gradient buffer + SGD pass (po_tree_sgd_step_range)")},
            "loss_first_last": [float(losses[0].item()), float(losses[-1].item())],
            "leaf_visits_per_step": visits / K,
            "roofline": {"bound": "hbm", "peak": peak, "unit": "GB/s", "peak_source": peak_src,
                         "alg_bytes_per_step": round(alg_survey),
                         "achieved": round(alg_survey / (t_max / K / 1e3) / 1e9, 1),
                         "frac": round(alg_survey / (t_max / K / 1e3) / 1e9 / peak, 4),
                         "alg_bytes_def": "SURVEY 8(d): visits*588 B (pass-1 and pass-2 record reads + 196 B "
                                          "gradient RMW) + nodes*2*32 B + rays*68 B",
                         "alg_bytes_as_implemented": round(alg),
                         "achieved_step": round(alg / (t_max / K / 1e3) / 1e9, 1),
                         "as_implemented_def": "visits*(4 sigma + 192 SH row + 196 gradient RMW) + nodes*32 + rays*68 "
                                               "(pass 2 replays 32-B stored segment records instead of re-reading "
                                               "the tree)"},
            "gpu_launches": int(launches), "clocks": clk,
            "e2e": {"value": round(e2e_value, 1), "unit": "rays/s",
                    "h2d_bytes_per_step": n_rays * (24 + 12) + (4 * ((n_rays + 31) // 32) if args.pass1_order == "costliest" else 0),
                    "d2h_bytes_per_step": 8, "entry": "OctreeOptimizer.train_from_host on pinned host batches (every step's "
                                                      "rays + targets (+ pass-1 group order) copied H2D on a side stream overlapping the "
                                                      "previous step; every step's loss copied D2H, async)"},
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def cpu_baseline(t_gen, seconds: float = 15.0, max_frames: int = 200):
    """The oracle as it stands, on this host's cores, on whole c1 frames (bounded by ~seconds)."""
    import numpy as np
    import gen
    import oracle
    oracle.build()
    ot = oracle.OracleTree(t_gen)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    frames = 0
    while frames < max_frames and (time.perf_counter() - t0) < seconds:
        cam, _, _ = gen.config_camera("c1", frames)
        rays = oracle.camera_rays(cam, W, H)
        oracle.render(ot, rays, gamma=GAMMA, nthreads=cores)
        frames += 1
    dt = time.perf_counter() - t0
    return {"value": round(frames / dt, 4), "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{frames} full c1 frames (views 0..{frames - 1}), ray generation + render, double precision, "
                      f"OpenMP {cores} threads, {dt:.1f} s"}


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    import gen
    t_gen = gen.scene_c1()
    # each step = a bounded sample of one c1 frame: every 4th pixel row (rows j = s mod 4),
    # 160,000 rays, ~0.1-0.3 s of CPU work; value is scaled to whole frames per second
    import oracle
    oracle.build()
    ot = oracle.OracleTree(t_gen)
    cores = os.cpu_count() or 1
    frac = 0.25

    def step(s):
        cam, _, _ = gen.config_camera("c1", s)
        rays = oracle.camera_rays(cam, W, H).reshape(H, W, 6)[s % 4::4].reshape(-1, 6)
        oracle.render(ot, rays, gamma=GAMMA, nthreads=cores)

    for s in range(args.warmup):
        step(s)
    t0 = time.perf_counter()
    for s in range(args.warmup, args.warmup + args.steps):
        step(s)
    dt = time.perf_counter() - t0
    v = frac * args.steps / dt
    sample = (f"{args.steps} steps x 1/4 of a c1 frame (every 4th row, 160k rays incl. ray generation), "
              f"double precision, OpenMP {cores} threads, {dt:.1f} s")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (procedural SDF scene, seeded)",
            "config": _workload_desc(t_gen) | {"parallelism": f"view-sharded x{ws}, tree replicated"},
            "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", choices=["c1", "c2", "c3", "c4", "c1thick", "c3sh25"], default="c1")
    ap.add_argument("--shard", choices=["view", "tile"], default="view",
                    help="c1/c3 at N>1: views per rank (weak) or the blocks of one view per rank (strong)")
    ap.add_argument("--views-per-launch", type=int, default=1,
                    help="render V consecutive orbit views per po_render launch (c2-style batches)")
    ap.add_argument("--l2", choices=["flush", "orbit", "same"], default="flush",
                    help="analysis only: 'orbit' = consecutive orbit views without flushing (warm, realistic "
                         "frame-to-frame reuse), 'same' = one view repeated; the reported number uses 'flush'")
    ap.add_argument("--flush", choices=["write+read", "write"], default="write+read",
                    help="L2 flush between timed steps (outside the timed region)")
    ap.add_argument("--rays", type=int, default=1 << 20, help="c4: rays per GPU per step")
    ap.add_argument("--reduce-scatter", action="store_true",
                    help="c4 at N>1: SGD fused into the gradient collective (reduce-scatter, shard update, all-gather)")
    ap.add_argument("--unfused-sgd", action="store_true",
                    help="c4 at N=1: separate gradient buffer + SGD pass instead of po_render_backward_sgd")
    ap.add_argument("--deterministic", action="store_true",
                    help="c4: order-fixed pass 2 (segmented reduction instead of atomics)")
    ap.add_argument("--max-seg", type=int, default=256,
                    help="c4: stored pass-1 segments per ray (0 = pass 2 re-traverses every ray)")
    ap.add_argument("--chunks", type=int, default=None,
                    help="c4: pass-2 chunks overlapped with the allreduce (default 4 if N>1, else 1)")
    ap.add_argument("--lr", type=float, default=3.0, help="c4: SGD learning rate (loss is a sum over rays)")
    ap.add_argument("--unsorted", action="store_true", help="c4: keep the sampled ray order (no Morton sort)")
    ap.add_argument("--pass1-order", choices=["costliest", "none"], default="costliest",
                    help="c4: order in which pass 1 claims the 32-ray groups (po_render_rays_ordered)")
    ap.add_argument("--ray-order", choices=["sampled", "leaf", "tileleaf"], default="tileleaf",
                    help="c4: keep the sampled order, sort the rays by first-entered leaf, or keep each 8x4 "
                         "tile's rays together and sort the tiles by their lowest first-entered leaf")
    ap.add_argument("--ray-sampling", choices=["tile", "pixel"], default="tile",
                    help="c4: sample 8x4 pixel tiles (coherent warps) or single pixels")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "c4":
        run_c4(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

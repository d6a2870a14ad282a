"""Where po_render_host's end-to-end time goes on c1 (measurement only): kernel alone, + H2D of
the camera, + image stores into mapped pinned host memory, and the synchronous host call."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2103_14024_b200 as po  # noqa: E402

t = gen.scene_c1()
tree = po.tree_from_gen(t)
recs = np.concatenate([gen.config_camera("c1", v)[0] for v in range(60)])
cams_host = torch.from_numpy(np.frombuffer(recs.tobytes(), np.float32).reshape(-1, 16).copy()).pin_memory()
cams_dev = cams_host.cuda()
dev_img = torch.empty((1, 800, 800, 3), device="cuda")
host_img = torch.empty((1, 800, 800, 3), pin_memory=True)
flush = torch.empty(64 << 20, device="cuda")
L = po.lib()
o = po._opts(0.01, (1.0, 1.0, 1.0))
cd = torch.empty((1, 16), device="cuda")


def run(mode, v):
    if mode == "kernel":
        po.po_render(tree, cams_dev[v:v + 1], 800, 800, out=dev_img)
    elif mode == "h2d+kernel":
        cd.copy_(cams_host[v:v + 1], non_blocking=True)
        po.po_render(tree, cd, 800, 800, out=dev_img)
    elif mode == "h2d+kernel->host":   # UVA: the pinned host pointer is the device pointer
        cd.copy_(cams_host[v:v + 1], non_blocking=True)
        po._check(L.po_render(tree.handle, po._ptr(cd), 1, 800, 800, ctypes.byref(o),
                              ctypes.c_void_p(host_img.data_ptr()), None))
    elif mode == "po_render_host":
        po.po_render_host(tree, cams_host.numpy()[v:v + 1], 800, 800, out_host=host_img.numpy())


for mode in ("kernel", "h2d+kernel", "h2d+kernel->host", "po_render_host"):
    ts = []
    for v in range(60):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(mode, v)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts = np.array(ts[10:])
    print(f"{mode:18s}: median {np.median(ts):6.1f} us  ({1e6 / np.median(ts):6.0f} FPS)")

"""Per-config CPU oracle baselines: the oracle as it stands (double precision,
OpenMP over rays) on this host's cores, 1 thread and all cores, for c0..c4.  Writes one JSON
object (stdout, and profiles/<tag>_oracle_baselines.json when a tag is given).  Test
infrastructure only: it times oracle/, the checker, never the product."""
import json
import os
import platform
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import oracle  # noqa: E402


def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor()


def timed(fn):
    t0 = time.perf_counter()
    fn()
    return time.perf_counter() - t0


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else None
    oracle.build()
    cores = os.cpu_count() or 1
    res = {"host": {"nproc": cores, "cpu": _cpu_model()}, "configs": {}}
    c0 = gen.scene_c0()
    ot0 = oracle.OracleTree(c0)
    cam, W, H = gen.config_camera("c0")
    r0 = oracle.camera_rays(cam, W, H)
    c1 = gen.scene_c1()
    ot1 = oracle.OracleTree(c1)
    for nt in (1, cores):
        key = f"{nt}_threads"
        d = {}
        # c0: full 64x64 view, recursive and brute force, + forward/backward at gamma 0
        s = timed(lambda: oracle.render(ot0, r0, gamma=0.01, nthreads=nt))
        d["c0_render_recursive"] = {"s": s, "Mrays_s": W * H / s / 1e6}
        s = timed(lambda: oracle.render(ot0, r0, gamma=0.01, mode=1, nthreads=nt))
        d["c0_render_bruteforce"] = {"s": s, "Mrays_s": W * H / s / 1e6}
        g = np.ones((r0.shape[0], 3))
        s = timed(lambda: oracle.backward(ot0, r0, g, gamma=0.0, nthreads=nt))
        d["c0_backward_gamma0"] = {"s": s, "Mrays_s": W * H / s / 1e6}
        # c1: one full 800x800 frame (ray generation + render)
        cam, W1, H1 = gen.config_camera("c1", 0)
        s = timed(lambda: oracle.render(ot1, oracle.camera_rays(cam, W1, H1), gamma=0.01, nthreads=nt))
        d["c1_frame"] = {"s": s, "fps": 1 / s, "Mrays_s": W1 * H1 / s / 1e6}
        # c2: 8 of the 200 orbit views, extrapolated to 200 (stated)
        t = 0.0
        for v in range(0, 200, 25):
            camv, _, _ = gen.config_camera("c2", v)
            t += timed(lambda: oracle.render(ot1, oracle.camera_rays(camv, W1, H1), gamma=0.01, nthreads=nt))
        d["c2_orbit"] = {"s_per_200_views_extrapolated": t * 25, "views_s": 8 / t, "sample": "views 0, 25, ..., 175"}
        # c4: 65,536-ray forward + backward subset at gamma 0 (one rank's batch is 1,048,576 rays)
        cams = gen.fibonacci_hemisphere(100, 4.0, 800, 800, 1111.111)
        rg = np.random.Generator(np.random.Philox(key=2))
        pick = rg.choice(100 * 800 * 800, size=65536, replace=False)
        rays = gen.camera_rays_f32(cams, 800, 800, pick // 640000, pick % 640000).astype(np.float64)
        gg = rg.normal(size=(65536, 3))
        s = timed(lambda: (oracle.render(ot1, rays, gamma=0.0, nthreads=nt),
                           oracle.backward(ot1, rays, gg, gamma=0.0, nthreads=nt)))
        d["c4_fwd_bwd"] = {"s_per_65536": s, "rays_s": 65536 / s,
                           "s_per_8M_extrapolated": s * 128, "note": "forward + backward, gamma 0"}
        res["configs"][key] = d
        print(key, json.dumps(d), flush=True)
    del ot1, c1
    c3 = gen.scene_c3()
    ot3 = oracle.OracleTree(c3)
    cam, W3, H3 = gen.config_camera("c3", 0)
    for nt in (1, cores):
        # c3 at one thread: one quarter of the frame (every 4th row), scaled (stated)
        rays = oracle.camera_rays(cam, W3, H3)
        frac = 0.25 if nt == 1 else 1.0
        sub = rays.reshape(H3, W3, 6)[::4].reshape(-1, 6) if nt == 1 else rays
        s = timed(lambda: oracle.render(ot3, sub, gamma=0.01, nthreads=nt))
        res["configs"][f"{nt}_threads"]["c3_frame"] = {"s": s / frac, "fps": frac / s, "Mrays_s": sub.shape[0] / s / 1e6,
                                                      "sample": "every 4th row, scaled" if nt == 1 else "full frame"}
    print(json.dumps(res))
    if tag:
        with open(os.path.join(ROOT, "profiles", f"{tag}_oracle_baselines.json"), "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

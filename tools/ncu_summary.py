#!/usr/bin/env python
"""Summarise ncu outputs from gpurun_out/ into profiles/ (committed evidence).

usage: python tools/ncu_summary.py <tag> [launches.csv] [prof.ncu-rep] [kernel]
writes profiles/<tag>_launches.md (per-kernel device time and share of the bench run),
profiles/<tag>_<kernel>_ncu.md (key --set full metrics) and, for k_render,
profiles/ncu_render_summary.json (dram bytes per launch, read by bench.py as `traffic`;
NCU_WORKLOAD=c2|c3 writes profiles/ncu_render_summary_<wl>.json instead).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct", "smsp__warp_issue_stalled_no_instruction_per_warp_active.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum", "local_load_bytes", "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum",
        "lts__t_sectors.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum",
        "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct", "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
        "smsp__warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]


def launches(path):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    ui = hdr.index("Metric Unit")
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        if r[ui] == "usecond":
            v *= 1e3
        elif r[ui] == "msecond":
            v *= 1e6
        name = r[ki].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    return tot, cnt


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (vals[i], units[i])
        d["Kernel Name"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        res.append(d)
    return res


def main():
    tag = sys.argv[1]
    lpath = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "launches.csv")
    rep = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", "prof_render.ncu-rep")
    kern = sys.argv[4] if len(sys.argv) > 4 else "k_render"
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if os.path.exists(lpath):
        tot, cnt = launches(lpath)
        all_ns = sum(tot.values())
        with open(os.path.join(ROOT, "profiles", f"{tag}_launches.md"), "w") as f:
            f.write(f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none, cold cache, serialised)\n\n")
            f.write("Command: `ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline`\n\n")
            f.write("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|\n")
            for k in sorted(tot, key=lambda k: -tot[k]):
                f.write(f"| `{k}` | {cnt[k]} | {tot[k] / 1e3:.1f} | {tot[k] / cnt[k] / 1e3:.2f} | {tot[k] / all_ns:.1%} |\n")
        print(open(os.path.join(ROOT, "profiles", f"{tag}_launches.md")).read())
    if os.path.exists(rep):
        res = raw(rep)
        with open(os.path.join(ROOT, "profiles", f"{tag}_{kern}_ncu.md"), "w") as f:
            f.write(f"# {tag}: ncu --set full of `{kern}` (--clock-control none)\n\n")
            for i, d in enumerate(res):
                f.write(f"## launch {i}: `{d['Kernel Name']}`\n\n| metric | value | unit |\n|---|---|---|\n")
                for k in KEYS:
                    if k in d:
                        f.write(f"| {k} | {d[k][0]} | {d[k][1]} |\n")
                f.write("\n")
        print(open(os.path.join(ROOT, "profiles", f"{tag}_{kern}_ncu.md")).read())
        if kern == "k_render" and res:
            d = res[-1]

            def mb(k):
                v, u = d[k]
                v = float(v.replace(",", ""))
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            by = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
            lts = mb("lts__t_bytes.sum") if "lts__t_bytes.sum" in d else None
            wl = os.environ.get("NCU_WORKLOAD", "c1")   # which bench workload the capture is of
            what = {"c1": "one c1 frame", "c2": "one c2 launch (200 views)", "c3": "one c3 frame"}.get(wl, wl)
            name = "ncu_render_summary.json" if wl == "c1" else f"ncu_render_summary_{wl}.json"
            json.dump({"dram_bytes_per_launch": by, "lts_bytes_per_launch": lts, "source": f"profiles/{tag}_{kern}_ncu.md (ncu --set full, {what}, cold L2)",
                       "duration": d["gpu__time_duration.sum"]},
                      open(os.path.join(ROOT, "profiles", name), "w"), indent=1)


if __name__ == "__main__":
    main()

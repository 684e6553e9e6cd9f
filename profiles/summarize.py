"""Summarise an ncu capture set (profiles/collect.sh) into tracked files under profiles/.

    python profiles/summarize.py r01        # reads gpurun_out/r01_*, writes profiles/r01_*

Writes:
  profiles/<tag>_launches.csv      the raw launch list (gpu__time_duration per launch)
  profiles/<tag>_summary.md        per-kernel share of the step + key --set full metrics
  profiles/traffic.json            DRAM bytes per launch per frame for bench.py's roofline
"""

from __future__ import annotations

import collections
import csv
import json
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "gpurun_out")
FRAMES = 16  # collect.sh profiles bench.py --frames 16 (the bench's own C4 batch)
LAP_ITERS = 10  # C4
BIL_ITERS = 5  # C4
# capture -> (name, frames in the launch)
CAPTURES = (("lap1", "laplacian_kernel_pass1", FRAMES), ("lap", "laplacian_kernel", FRAMES),
            ("tri", "triangulate_kernel", FRAMES), ("bil", "bilateral_kernel", FRAMES),
            ("bil1", "bilateral_kernel_iter1", FRAMES), ("qx", "quad_extras_kernel (C3)", 512),
            ("lap64", "laplacian_f64_kernel (strict)", FRAMES),
            ("bil64", "bilateral_f64_kernel (strict)", FRAMES))

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
    "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return {}
    h, u, v = rows[0], rows[1], rows[2]
    d = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else "?"}
    for m in METRICS:
        if m in h:
            i = h.index(m)
            d[m] = (v[i], u[i])
    stalls = {}
    for i, name in enumerate(h):
        if name.startswith("smsp__average_warps_issue_stalled_") and \
                name.endswith("_per_issue_active.ratio"):
            try:
                stalls[name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v[i])
            except ValueError:
                pass
    d["stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
    return d


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
            if name == "bilateral_packed_kernel":
                name = "bilateral_kernel"  # one bench stage: iteration 1 + packed 2..B
            if name == "laplacian3p_kernel" or name == "laplacian3_kernel":
                name = "laplacian_kernel"  # one bench stage: pass 1 + packed passes 2..L
            agg[name].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    return {k: (len(v), sum(v) / len(v), sum(v) / tot) for k, v in agg.items()}


def main(tag):
    lines = [f"# ncu summary {tag}", "",
             "Command: `python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "
             f"--no-strict --frames {FRAMES}` (1080x1920, lap 10 + bil 5; 16 frames = the "
             "bench's own batch, inputs 398 MB > L2).  Launch-list times are "
             "cold-cache and serialised: compare SHARES with bench.py's stage times.", ""]
    lp = os.path.join(OUT, f"{tag}_launches.csv")
    if os.path.exists(lp):
        shutil.copy(lp, os.path.join(HERE, f"{tag}_launches.csv"))
        lines += ["## Launch list (all launches of the command)", "",
                  "| kernel | launches | mean us | share |", "|---|---|---|---|"]
        for k, (n, mean, share) in sorted(launch_shares(lp).items(), key=lambda kv: -kv[1][2]):
            lines.append(f"| {k} | {n} | {mean / 1e3:.1f} | {share:.3f} |")
        lines.append("")
    traffic = {}
    for short, kname, frames in CAPTURES:
        rep = os.path.join(OUT, f"{tag}_{short}.ncu-rep")
        if not os.path.exists(rep):
            continue
        d = raw_metrics(rep)
        if "dram__bytes_read.sum" not in d:
            continue
        lines += [f"## {kname} (`--set full`, one launch, {frames} frames)", "",
                  f"`{d.get('kernel', '?')[:140]}`", "", "| metric | value |", "|---|---|"]
        for m in METRICS:
            if m in d:
                lines.append(f"| {m} | {d[m][0]} {d[m][1]} |")
        lines.append(f"| top stalls (cycles per issue) | "
                     f"{', '.join(f'{k} {v:.2f}' for k, v in d['stalls'].items())} |")
        lines.append("")
        unit = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rb = float(d["dram__bytes_read.sum"][0]) * unit[d["dram__bytes_read.sum"][1]]
        wb = float(d["dram__bytes_write.sum"][0]) * unit[d["dram__bytes_write.sum"][1]]
        traffic[kname] = {"dram_bytes_per_launch_per_frame": (rb + wb) / frames,
                          "dram_read_bytes": rb, "dram_write_bytes": wb, "frames": frames,
                          "capture": f"profiles/{tag}_summary.md"}
    if "bilateral_kernel_iter1" in traffic and "bilateral_kernel" in traffic:
        # the bench's bilateral "launch" is the stage / B: iteration 1 + (B-1) packed ones
        b1 = traffic.pop("bilateral_kernel_iter1")
        bp = traffic["bilateral_kernel"]
        bp["dram_bytes_per_launch_per_frame"] = (
            b1["dram_bytes_per_launch_per_frame"] + (BIL_ITERS - 1) * bp["dram_bytes_per_launch_per_frame"]
        ) / BIL_ITERS
        bp["note"] = f"mean over the {BIL_ITERS} launches: iteration 1 + {BIL_ITERS - 1} packed"
        bp["iteration1_bytes_per_frame"] = b1["dram_bytes_per_launch_per_frame"]
    if "laplacian_kernel_pass1" in traffic and "laplacian_kernel" in traffic:
        l1 = traffic.pop("laplacian_kernel_pass1")
        lp = traffic["laplacian_kernel"]
        lp["dram_bytes_per_launch_per_frame"] = (
            l1["dram_bytes_per_launch_per_frame"] + (LAP_ITERS - 1) * lp["dram_bytes_per_launch_per_frame"]
        ) / LAP_ITERS
        lp["note"] = f"mean over the {LAP_ITERS} launches: pass 1 + {LAP_ITERS - 1} packed"
        lp["pass1_bytes_per_frame"] = l1["dram_bytes_per_launch_per_frame"]
    with open(os.path.join(HERE, f"{tag}_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(HERE, "traffic.json"), "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")

"""Summarise profiles/collect_precise.sh captures into profiles/<tag>_precise_summary.md
(and copy the launch lists): python profiles/summarize_precise.py <tag>"""
import collections
import csv
import os
import shutil
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize import HERE, METRICS, OUT, raw_metrics  # noqa: E402

KERNELS = (("lap", "Laplacian pass (laplacian_f64_tma_kernel<3, MIXED>)"),
           ("fc", "FC data (fc_rows_kernel)"),
           ("bil", "bilateral iteration (strict: bilateral_f64s_kernel; mixed: bilateral_kernel "
                   "iteration 1 -- from the f64 grid since r02o, from the FC arrays before)"))


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0].replace("void ", "").split("::")[-1].split("<")[0]
            agg[name].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot:.3f} |")
    return out


def main(tag):
    lines = [f"# ncu summary {tag}: strict and mixed precision chains", "",
             "Command: `python profiles/strict_driver.py --frames 16 --steps 2 --precision "
             "strict|mixed` (C4 1080x1920, lap 10 + bil 5, 16 frames, eager launches).  "
             "Launch-list times are cold-cache and serialised.", ""]
    for p in ("strict", "mixed"):
        lp = os.path.join(OUT, f"{tag}_{p}_launches.csv")
        if os.path.exists(lp):
            shutil.copy(lp, os.path.join(HERE, f"{tag}_{p}_launches.csv"))
            lines += [f"## {p}: launch list (2 steps)", ""] + launch_table(lp) + [""]
        for short, title in KERNELS:
            rep = os.path.join(OUT, f"{tag}_{p}_{short}.ncu-rep")
            if not os.path.exists(rep):
                continue
            d = raw_metrics(rep)
            if "dram__bytes_read.sum" not in d:
                continue
            lines += [f"### {p}: {title}", "", f"`{d.get('kernel', '?')[:140]}`", "",
                      "| metric | value |", "|---|---|"]
            for m in METRICS:
                if m in d:
                    lines.append(f"| {m} | {d[m][0]} {d[m][1]} |")
            lines.append(f"| top stalls (cycles per issue) | "
                         f"{', '.join(f'{k} {v:.2f}' for k, v in d['stalls'].items())} |")
            lines.append("")
    with open(os.path.join(HERE, f"{tag}_precise_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")

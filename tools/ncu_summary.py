#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum) and an
`ncu --set full` report into profiles/<tag>_*.md / .json (run here, no GPU).

    python tools/ncu_summary.py <tag> [launches.csv] [prof.ncu-rep] [--config C5 --prec 32]
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6,
         "ns": 1e-9, "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9}


def short(name):
    return name.split("(")[0].split("<")[0].replace("void ", "").replace("vx::", "").strip()


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"]) * SCALE.get(d["Metric Unit"], 1)
            out.append((short(d["Kernel Name"]), v))
    return out


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                try:
                    d[k] = float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    d[k] = r[i]
        res.append(d)
    return res


def main():
    tag = sys.argv[1]
    lc = sys.argv[2] if len(sys.argv) > 2 else f"gpurun_out/launches_{tag}.csv"
    rep = sys.argv[3] if len(sys.argv) > 3 else f"gpurun_out/prof_{tag}.ncu-rep"
    nvox = 512 * 256 * 256
    alg = {"k_bonds": 164, "k_integrate": 220, "k_step_fused": 112}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    md = [f"# ncu summary `{tag}` (C5 512x256x256 fp32, one B200)\n"]
    if os.path.exists(lc):
        L = launches(lc)
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for k, v in L:
            tot[k] += v
            cnt[k] += 1
        allt = sum(tot.values())
        md.append("## Launch list (cold-cache, serialised; compare shares)\n")
        md.append("| kernel | launches | mean ms | share of all |\n|---|---|---|---|")
        for k in sorted(tot, key=tot.get, reverse=True):
            md.append(f"| {k} | {cnt[k]} | {1e3 * tot[k] / cnt[k]:.4f} | {tot[k] / allt:.3f} |")
        step = [k for k in tot if k in alg or k == "k_clock"]
        st = sum(tot[k] for k in step)
        md.append("\nPer-step kernels only (clock, bonds, integrate / fused):\n")
        for k in step:
            md.append(f"- {k}: {tot[k] / st:.3f} of the step")
        json.dump({"launches": L}, open(os.path.join(ROOT, "profiles", f"{tag}_launches.json"), "w"),
                  indent=1)
    traffic = {}
    if os.path.exists(rep):
        F = full(rep)
        md.append("\n## `ncu --set full` (per launch)\n")
        md.append("| kernel | ms | DRAM read GB | DRAM write GB | B/voxel | alg B/voxel | DRAM % peak | "
                  "SM % | warps active % | regs |\n|---|---|---|---|---|---|---|---|---|---|")
        for d in F:
            t = d.get("gpu__time_duration.sum", 0)
            rd = d.get("dram__bytes_read.sum", 0)
            wr = d.get("dram__bytes_write.sum", 0)
            md.append(f"| {d['kernel']} | {1e3 * t:.4f} | {rd / 1e9:.3f} | {wr / 1e9:.3f} | "
                      f"{(rd + wr) / nvox:.1f} | {alg.get(d['kernel'], '-')} | "
                      f"{d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                      f"{d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                      f"{d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                      f"{d.get('launch__registers_per_thread', 0):.0f} |")
            name = {"k_bonds": "bonds", "k_integrate": "integrate", "k_step_fused": "fused"}.get(
                d["kernel"])
            if name:
                traffic[f"C5:fp32:{name}"] = rd + wr
        json.dump(F, open(os.path.join(ROOT, "profiles", f"{tag}_full.json"), "w"), indent=1)
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        old = json.load(open(tp)) if os.path.exists(tp) else {}
        old.update(traffic)
        old["_source"] = f"profiles/{tag}_full.json (ncu --set full, dram__bytes_read+write per launch)"
        json.dump(old, open(tp, "w"), indent=1)
    open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w").write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Per-source-line dynamic instruction counts (and the MOVs among them) of one
kernel from an ncu report: python tools/ncu_lines.py <rep> [voxels] [top]"""
import collections, csv, io, re, subprocess, sys
rep = sys.argv[1]
vox = float(sys.argv[2]) if len(sys.argv) > 2 else 33554432.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file, hdr, cur_line = None, None, None
agg = {}
movs = collections.Counter()
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0].isdigit():
        cur_line = (cur_file, int(r[0]), r[1].strip()[:80])
        d = dict(zip(hdr[4:], r[4:]))
        try:
            agg[cur_line] = (float(r[hdr.index("Instructions Executed")] or 0),
                             float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0))
        except ValueError:
            pass
    elif r[0] == "" and cur_line and len(r) > 7:
        src = r[3]
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", src.strip())
        try:
            n = float(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        if m and m.group(2) in ("MOV", "IMAD") and (m.group(2) == "MOV" or ".MOV" in src):
            movs[cur_line] += n
tot = sum(v[0] for v in agg.values())
stot = sum(v[1] for v in agg.values()) or 1
print(f"total {32 * tot / vox:.1f} thread-inst / voxel")
for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{32 * n / vox:6.1f} mov {32 * movs[k] / vox:5.1f} stall {100 * s / stot:4.1f}%  {k[0]}:{k[1]} {k[2]}")
print(f"moves total {32 * sum(movs.values()) / vox:.1f}")
for k, n in movs.most_common(25):
    print(f"  mov {32 * n / vox:5.1f}  {k[0]}:{k[1]} {k[2]}")

#!/usr/bin/env python
"""Dynamic SASS opcode histogram of one kernel from an ncu report (source page,
`Instructions Executed` per SASS line), per voxel-thread.
   python tools/sass_dyn.py <report.ncu-rep> [voxels] [kernel-substring]"""
import collections, csv, io, re, subprocess, sys
rep = sys.argv[1]
vox = float(sys.argv[2]) if len(sys.argv) > 2 else 33554432.0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
iE = hdr.index("Instructions Executed")
iS = hdr.index("Source")
iW = hdr.index("Warp Stall Sampling (All Samples)")
ops = collections.Counter()
stall = collections.Counter()
tot = 0
lines = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    n = float(r[iE] or 0)
    src = r[iS].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.\S+)?", src)
    if not m:
        continue
    op = m.group(2)
    ops[op] += n
    stall[op] += float(r[iW] or 0)
    tot += n
    lines.append((n, float(r[iW] or 0), src))
print(f"total warp-inst {tot:.4g}  per voxel {tot / vox:.3f}  (x32 = {32 * tot / vox:.1f} thread-inst / voxel)")
tstall = sum(stall.values())
for op, n in ops.most_common(45):
    print(f"{op:10s} {32 * n / vox:7.1f} /voxel  {100 * n / tot:5.1f}%   stall {100 * stall[op] / tstall:5.1f}%")

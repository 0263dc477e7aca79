#!/usr/bin/env python
"""Static SASS instructions (and MOVs) per source line of one kernel (no GPU):
   python tools/sass_lines.py <kernel-substring> [lib] [top]"""
import collections, re, subprocess, sys
pat = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_1212_2845_b200/libvoxsim.so"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
import os, tempfile
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cub = [os.path.join(tmp, x) for x in os.listdir(tmp) if x.endswith(".cubin")][0]
out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*\.text\.", out)
for f in funcs[1:]:
    name = f.split(":", 1)[0].strip()
    if pat not in name:
        continue
    cur = None
    tot = collections.Counter(); mov = collections.Counter()
    for line in f.split("\n"):
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", line)
        if m and cur:
            tot[cur] += 1
            if m.group(2) == "MOV" or (m.group(2) == "IMAD" and (m.group(3) or "").startswith(".MOV")):
                mov[cur] += 1
    print(name, sum(tot.values()), "instr,", sum(mov.values()), "moves")
    for k, v in mov.most_common(top):
        print(f"  {v:4d} mov / {tot[k]:4d}  {k[0]}:{k[1]}")
    break

#!/usr/bin/env python
"""Static SASS opcode histogram of one kernel in libvoxsim.so (no GPU needed).
   python tools/sass_hist.py <kernel-substring> [lib]"""
import collections, re, subprocess, sys
pat = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_1212_2845_b200/libvoxsim.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ops = collections.Counter()
    for line in f.split("\n"):
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m:
            ops[m.group(2).split(".")[0]] += 1
    print(name, "total", sum(ops.values()))
    print("  ", ", ".join(f"{k} {v}" for k, v in ops.most_common(40)))

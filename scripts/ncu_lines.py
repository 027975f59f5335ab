"""Aggregate an ncu source page (cuda,sass) by (file, line), per kernel (dev tool).
usage: ncu_lines.py REPORT [TOP] [KERNEL-SUBSTRING]"""
import csv
import os
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
want = sys.argv[3] if len(sys.argv) > 3 else ""
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
srcs = {}


def src_line(path, ln):
    if path not in srcs:
        srcs[path] = open(path).read().split("\n") if os.path.exists(path) else []
    L = srcs[path]
    return L[ln - 1].strip()[:70] if 0 < ln <= len(L) else ""


path, fn, hdr, per = None, None, None, {}
for r in csv.reader(txt.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        path = r[1]
        continue
    if len(r) == 2 and r[0] == "Function Name":
        fn = r[1][:100]
        per.setdefault(fn, [])
        continue
    if len(r) > 5 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and fn and len(r) == len(hdr) and r[2] == "-":
        d = dict(zip(hdr, r))
        try:
            per[fn].append((os.path.basename(path), int(d["Line No"]), int(d["Warp Stall Sampling (All Samples)"]),
                            int(d["Instructions Executed"]), path))
        except ValueError:
            pass
for fn, out in per.items():
    if want not in fn:
        continue
    ts = sum(o[2] for o in out) or 1
    ti = sum(o[3] for o in out) or 1
    print(f"== {fn}\n   samples {ts} warp-instr {ti}")
    for f, ln, s, i, pth in sorted(out, key=lambda o: -o[3 if len(sys.argv) < 5 else 2])[:top]:
        print(f"{f[:14]:14s}{ln:5d} samp {100*s/ts:5.1f}% inst {100*i/ti:5.1f}%  {src_line(pth, ln)}")

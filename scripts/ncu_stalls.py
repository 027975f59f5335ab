"""Per-source-line stall breakdown of one kernel in an ncu report (dev tool).
usage: ncu_stalls.py REPORT KERNEL [TOP]"""
import csv
import os
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "-k", kern,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
src = {}
path = None
hdr = None
agg = defaultdict(lambda: defaultdict(float))
cur = None
for r in csv.reader(txt.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        path = r[1]
        continue
    if len(r) > 5 and r[0] in ("Line No", "Address"):
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if "Line No" in d and d.get("Address") == "-" or (d.get("Line No", "").isdigit() and d.get("Address", "-") == "-"):
        cur = (path, int(d["Line No"]))
        continue
    if cur is None:
        continue
    for k, v in d.items():
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                agg[cur][k[6:]] += float(v)
            except ValueError:
                pass
tot = sum(sum(v.values()) for v in agg.values()) or 1
bytype = defaultdict(float)
for v in agg.values():
    for k, x in v.items():
        bytype[k] += x
print("stall totals:", ", ".join(f"{k} {100*x/tot:.1f}%" for k, x in sorted(bytype.items(), key=lambda t: -t[1])[:8]))


def line(p, n):
    if p not in src:
        src[p] = open(p).read().split("\n") if p and os.path.exists(p) else []
    L = src[p]
    return L[n - 1].strip()[:60] if 0 < n <= len(L) else ""


for (p, n), v in sorted(agg.items(), key=lambda t: -sum(t[1].values()))[:top]:
    s = sum(v.values())
    parts = ", ".join(f"{k} {100*x/tot:.1f}" for k, x in sorted(v.items(), key=lambda t: -t[1])[:3] if x > 0)
    print(f"{os.path.basename(p or '')[:12]:12s}{n:5d} {100*s/tot:5.1f}% [{parts}]  {line(p, n)}")

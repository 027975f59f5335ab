"""Per source line of one kernel: stall-reason samples (dev tool).
usage: ncu_stall_lines.py REPORT KERNEL-SUBSTRING [TOP] [LINE_LO LINE_HI]"""
import csv
import subprocess
import sys

rep, want = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"], capture_output=True,
                     text=True).stdout
path = fn = hdr = None
rows = []
tot = {}
for r in csv.reader(txt.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if len(r) == 2 and r[0] in ("Function Name", "File Name"):
        if r[0] == "Function Name":
            fn = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or fn is None or want not in fn or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if not d["Line No"]:
        continue
    try:
        samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    except ValueError:
        continue
    st = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "(Not Issued)" not in k and v.isdigit()}
    for k, v in st.items():
        tot[k] = tot.get(k, 0) + v
    rows.append((samp, path, d["Line No"], d["Source"][:60], st))
T = sum(x[0] for x in rows) or 1
print("total samples", T, " by reason:", ", ".join(f"{k}={100 * v / T:.1f}%" for k, v in
                                                   sorted(tot.items(), key=lambda kv: -kv[1]) if v))
for samp, p, ln, src, st in sorted(rows, key=lambda x: -x[0])[:top]:
    reasons = ", ".join(f"{k}={v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
    print(f"{p:14s}{ln:>5s} {100 * samp / T:5.1f}%  {src:60s} {reasons}")

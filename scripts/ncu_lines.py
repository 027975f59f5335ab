"""Aggregate an ncu source page (cuda,sass) by CUDA source line (dev tool)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else "paper_2603_21444_b200/csrc/spgemm.cu"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
lines = open(src).read().split("\n")
rows = list(csv.reader(txt.splitlines()))
hdr, out = None, []
for r in rows:
    if len(r) > 5 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        d = dict(zip(hdr, r))
        try:
            out.append((int(d["Line No"]), int(d["Warp Stall Sampling (All Samples)"]), int(d["Instructions Executed"])))
        except ValueError:
            pass
ts = sum(o[1] for o in out) or 1
ti = sum(o[2] for o in out) or 1
print(f"samples {ts} warp-instr {ti}")
for ln, s, i in sorted(out, key=lambda o: -o[1])[:top]:
    print(f"{ln:5d} samp {100*s/ts:5.1f}% inst {100*i/ti:5.1f}%  {lines[ln-1].strip()[:80] if ln <= len(lines) else ''}")

"""Top SASS instructions of one kernel in an ncu report (dev tool).
usage: ncu_sass.py REPORT KERNEL-REGEX [TOP] [launch-skip]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "-k", f"regex:{kre}",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
hdr, out, seen = None, [], set()
for r in csv.reader(txt.splitlines()):
    if len(r) > 5 and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Address"] in seen:
            continue
        seen.add(d["Address"])
        try:
            out.append((int(d["Instructions Executed"]), int(d["Warp Stall Sampling (All Samples)"]),
                        d["Address"][-5:], d["Source"].strip()[:70]))
        except ValueError:
            pass
ti = sum(o[0] for o in out) or 1
ts = sum(o[1] for o in out) or 1
print(f"sass {len(out)} inst {ti} samples {ts}")
key = 0 if len(sys.argv) > 5 else 1
for o in sorted(out, key=lambda o: -o[key])[:top]:
    print(f"{o[2]} inst {o[0]:11d} ({100*o[0]/ti:4.1f}%) samp {100*o[1]/ts:4.1f}%  {o[3]}")

"""Writes profiles/traffic.json from an `ncu --set full` capture of the
numeric kernel (dev tool): dram__bytes_read.sum + dram__bytes_write.sum of
the launch, keyed by config and tied to the kernel source it was captured on
(sha256 of paper_2603_21444_b200/csrc/spgemm.cu; bench.py reports it only
while the source is unchanged). usage: ncu_traffic.py REPORT [config_n1]"""
import csv
import hashlib
import io
import json
import os
import subprocess
import sys

rep = sys.argv[1]
key = sys.argv[2] if len(sys.argv) > 2 else "config2_n1"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
m = dict(zip(hdr, vals))
u = dict(zip(hdr, units))


def num(k):
    v = float(m[k].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "second": 1.0, "s": 1.0}.get(u[k], 1.0)
    return v * scale


rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
sha = hashlib.sha256(open(os.path.join(root, "paper_2603_21444_b200", "csrc", "spgemm.cu"), "rb").read()).hexdigest()
path = os.path.join(root, "profiles", "traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d = {k: v for k, v in d.items() if isinstance(v, dict)}
d[key] = {"bytes": int(rd + wr), "read_bytes": int(rd), "write_bytes": int(wr),
          "kernel": m.get("Kernel Name", ""), "duration_s": num("gpu__time_duration.sum"),
          "spgemm_cu_sha16": sha[:16], "report": os.path.basename(rep)}
json.dump(d, open(path, "w"), indent=1)
print(json.dumps(d[key]))

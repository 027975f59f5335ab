"""Per-pull timing of the trident exchange (dev tool): config 2 (ER 2^22,
16/row, C = A*A) through the single-process driver with P ranks on the
visible GPUs; prints every measured transfer event (bytes, duration, GB/s).
usage: exchange_probe.py P LAMBDA [reps]"""
import sys
import time
sys.path.insert(0, ".")
import paper_2603_21444_b200 as spg  # noqa: E402

P, lam = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
a = spg.gen_erdos_renyi(1 << 22, 16.0 / (1 << 22), 1)
grid = spg.TridentGrid.create(P, lam)
for it in range(reps):
    t0 = time.perf_counter()
    r = spg.trident_spgemm(a, a, grid)
    wall = time.perf_counter() - t0
    ev = [e for e in r.events if e["type"] in ("transfer-complete", "allgather-complete")]
    print(f"rep {it}: wall {wall:.2f} s, {len(ev)} pulls / allgathers; per-rank exchange ms "
          f"{[round(float(x), 3) for x in r.timeline[:, :, 0].sum(axis=1)]}")
    if it == reps - 1:
        for e in sorted(ev, key=lambda e: (e.get("dst", -1), e["t_start"])):
            d = (e["t_end"] - e["t_start"]) * 1e3
            who = f"dst {e['dst']} src {e['src']}" if "dst" in e else f"actors {e.get('actors')}"
            print(f"  {e['type'][:9]} {who} {e['operand']} bytes {e['bytes']:>11} "
                  f"t {e['t_start'] * 1e3:8.3f}..{e['t_end'] * 1e3:8.3f} ms  {d:7.3f} ms  {e['bytes'] / max(d, 1e-9) / 1e6:7.1f} GB/s")

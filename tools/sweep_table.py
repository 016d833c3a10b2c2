"""Table of ring_sweep JSON lines: ms, wire GB/s and fraction of the 770 GB/s
NVLink peak per (p, CTAs, n, codec), NCCL beside it."""
import json
import sys

rows, lag = [], None
for f in sys.argv[1:]:
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            if "lag" in d and "codec" not in d:
                lag = d["lag"]
                continue
            d["lag"] = lag
            rows.append(d)
nccl = {(r["p"], r["n"]): r["ms"] for r in rows if r["codec"] == "nccl"}
print(f"{'lag':>4} {'p':>2} {'ctas':>5} {'n':>10} {'codec':>8} {'ms':>8} {'wire GB/s':>10} {'frac':>6} {'nccl ms':>8} ok")
for r in rows:
    if r["codec"] == "nccl":
        continue
    print(f"{str(r['lag']):>4} {r['p']:>2} {r.get('ctas', 0):>5} {r['n']:>10} {r['codec']:>8} {r['ms']:8.4f} {r['wire_busbw_gbs']:10.1f} "
          f"{r['wire_busbw_gbs'] / 770:6.3f} {nccl.get((r['p'], r['n']), float('nan')):8.4f} "
          f"{r.get('replicas_bit_identical', '')}")

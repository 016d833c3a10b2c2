"""Table of ring_sweep JSON lines per library variant: python tools/variant_table.py DIR v1 v2 ..."""
import json
import sys

O, vs = sys.argv[1], sys.argv[2:]
for np_ in (2, 4):
    d, nccl, bad = {}, {}, set()
    for v in vs:
        try:
            for l in open(f"{O}/p{np_}_{v}.jsonl"):
                r = json.loads(l)
                if r["codec"] == "nccl":
                    nccl[r["n"]] = r["ms"] * 1e3
                else:
                    d[(r["n"], r["codec"], v)] = r["ms"] * 1e3
                    if r.get("replicas_bit_identical") is False:
                        bad.add((r["n"], r["codec"], v))
        except FileNotFoundError:
            pass
    if not d:
        continue
    print(f"p = {np_}: n codec " + " ".join(f"{v:>10s}" for v in vs) + "      nccl")
    for n in sorted({k[0] for k in d}):
        for c in ("none", "trunc16", "quant8"):
            cells = [d.get((n, c, v), float("nan")) for v in vs]
            flag = " MISMATCH" if any((n, c, v) in bad for v in vs) else ""
            print(f"  {n:>9} {c:8s}" + " ".join(f"{t:10.1f}" for t in cells) + f"  {nccl.get(n, float('nan')):8.1f}{flag}")

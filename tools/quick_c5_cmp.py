"""Compare two quick ring sweeps (tools/r02_quick_c5.sh outputs): us per call and NCCL."""
import json
import sys

a, b = sys.argv[1], sys.argv[2]
for np_ in (2, 4):
    def load(d):
        try:
            return [json.loads(l) for l in open(f"{d}/p{np_}.jsonl")]
        except FileNotFoundError:
            return []
    ra, rb = load(a), load(b)
    nccl = {r["n"]: r["ms"] for r in rb if r.get("codec") == "nccl"}
    old = {(r["n"], r["codec"]): r["ms"] for r in ra}
    print(f"p = {np_}: n codec  before_us  after_us  nccl_us  after/nccl")
    for r in rb:
        if r.get("codec") in ("none", "trunc16", "quant8"):
            o = old.get((r["n"], r["codec"]))
            print(f"  {r['n']:>10} {r['codec']:8s} {o * 1e3 if o else float('nan'):8.1f} {r['ms'] * 1e3:8.1f} "
                  f"{nccl.get(r['n'], 0) * 1e3:8.1f}  {r['ms'] / nccl.get(r['n'], 1):.2f}")

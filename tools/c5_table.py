"""Markdown table of a tools/c5_sweep.sh log: us and fp32-equivalent busbw
per size x codec x p, NCCL fp32 beside it."""
import json
import sys

rows = [json.loads(ln) for ln in open(sys.argv[1]) if ln.startswith("{")]
for p in sorted({r["p"] for r in rows}):
    print(f"\n### p = {p}\n")
    print("| n (fp32 elems) | bytes | none us (GB/s) | trunc16 us (GB/s) | quant8 us (GB/s) | NCCL fp32 us (GB/s) |")
    print("|---|---|---|---|---|---|")
    by = {}
    for r in rows:
        if r["p"] == p:
            by.setdefault(r["n"], {})[r["codec"]] = r
    for n in sorted(by):
        c = by[n]
        cell = [f"{c[k]['ms'] * 1e3:.1f} ({c[k]['busbw_gbs']:.0f})" if k in c else "-"
                for k in ("none", "trunc16", "quant8", "nccl")]
        b = 4 * n
        h = f"{b / 2**30:.0f} GiB" if b >= 2**30 else f"{b / 2**20:.0f} MiB" if b >= 2**20 else f"{b / 2**10:.0f} KiB" if b >= 1024 else f"{b} B"
        print(f"| {n} | {h} | " + " | ".join(cell) + " |")

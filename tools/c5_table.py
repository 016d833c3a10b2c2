"""Markdown tables of a tools/c5_sweep.sh run: per size x codec x p the
device time, fp32-equivalent busbw and wire fraction of NVLink (770 GB/s),
NCCL fp32 beside it, the Eq. 5 prediction (pred / measured, 25 % flag) and
the reference's CPU ring (ms, speed-up). Clock records summarised."""
import json
import sys

rows = []
for f in sys.argv[1:]:
    rows += [json.loads(ln) for ln in open(f) if ln.startswith("{")]
sym = [r for r in rows if "eq5_symbols" in r]
rows = [r for r in rows if "codec" in r]
for s in sym:
    e = s["eq5_symbols"]
    print(f"Eq. 5 symbols: alpha {e.get('alpha_s', 0) * 1e6:.2f} us, beta push {e.get('push_gbs', 0):.0f} GB/s, "
          f"S {e['S_s'] * 1e6:.2f} us; host {s.get('cpu')} ({s.get('cpu_count')} cpus)")
clk = [r["clocks"] for r in rows if r.get("clocks")]
if clk:
    mhz = sorted(c["sm_mhz"] for c in clk if c.get("sm_mhz"))
    reasons = sorted({x for c in clk for x in c.get("reasons", [])})
    print(f"\nclocks: {len(clk)} series, SM {mhz[0]:.0f}-{mhz[-1]:.0f} MHz (max {clk[0].get('sm_max_mhz')}), "
          f"throttle reasons: {reasons or 'none'}")
for p in sorted({r["p"] for r in rows}):
    print(f"\n### p = {p}\n")
    print("| n | bytes | codec | us | fp32-eq GB/s | wire frac | NCCL us | Eq. 5 us (pred/meas) | Eq. 5 ext us (pred/meas) "
          "| CPU ref ms (x) |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    by = {}
    for r in rows:
        if r["p"] == p:
            by.setdefault(r["n"], {})[r["codec"]] = r
    for n in sorted(by):
        c = by[n]
        b = 4 * n
        h = (f"{b / 2**30:.0f} GiB" if b >= 2**30 else f"{b / 2**20:.0f} MiB" if b >= 2**20
             else f"{b / 2**10:.0f} KiB" if b >= 1024 else f"{b} B")
        nccl = f"{c['nccl']['ms'] * 1e3:.1f}" if "nccl" in c else "-"
        for k in ("none", "trunc16", "quant8"):
            if k not in c:
                continue
            r = c[k]
            e = r.get("eq5")
            eq = f"{e['eq5_ms'] * 1e3:.1f} ({e['eq5_over_measured']:.2f}{'*' if e['flagged'] else ''})" if e else "-"
            ex = (f"{e['eq5_ext_ms'] * 1e3:.1f} ({e['eq5_ext_over_measured']:.2f}{'*' if e['ext_flagged'] else ''})"
                  if e and "eq5_ext_ms" in e else "-")
            cpu = r.get("cpu_reference")
            cp = f"{cpu['ms']:.1f} ({cpu['speedup']:.0f}x)" if cpu else "-"
            print(f"| {n} | {h} | {k} | {r['ms'] * 1e3:.1f} | {r['busbw_gbs']:.0f} | {r['wire_busbw_gbs'] / 770:.2f} | "
                  f"{nccl} | {eq} | {ex} | {cp} |")
print("\n`*` = Eq. 5 off by more than the reference's 25 % flag (harness.py:687-720).")

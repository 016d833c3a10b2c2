"""Markdown table of a run_matrix.sh output directory (one bench JSON per cell)."""
import json
import os
import sys

ROWS = [("c1_pipe", "C1 MNIST MLP, none", "Pipe-SGD width 2 (graphs)"),
        ("c1_sync", "C1 MNIST MLP, none", "D-Sync width 1 (graphs)"),
        ("c2_pipe", "C2 CIFAR CNN, trunc16", "Pipe-SGD width 2 (graphs)"),
        ("c2_pipe_eager", "C2 CIFAR CNN, trunc16", "Pipe-SGD width 2 (eager)"),
        ("c2_sync", "C2 CIFAR CNN, trunc16", "D-Sync width 1 (graphs)"),
        ("c2_sync_eager", "C2 CIFAR CNN, trunc16", "D-Sync width 1 (eager)"),
        ("c2_ps", "C2 CIFAR CNN, trunc16", "PS-Sync (eager)"),
        ("c3_pipe", "C3 AlexNet, quant8", "Pipe-SGD width 2 (graphs)"),
        ("c3_pipe_eager", "C3 AlexNet, quant8", "Pipe-SGD width 2 (eager)"),
        ("c3_sync", "C3 AlexNet, quant8", "D-Sync width 1 (graphs)"),
        ("c3_sync_eager", "C3 AlexNet, quant8", "D-Sync width 1 (eager)"),
        ("c3_ps", "C3 AlexNet, quant8", "PS-Sync (eager)"),
        ("c4_pipe", "C4 ResNet-50, none", "Pipe-SGD width 2 (graphs)"),
        ("c4_sync", "C4 ResNet-50, none", "D-Sync width 1 (graphs)")]


def load(d, name):
    p = os.path.join(d, name + ".json")
    if not os.path.exists(p):
        return None
    ls = [ln for ln in open(p) if ln.startswith("{")]
    return json.loads(ls[-1]) if ls else None


def main(d):
    print("| config | scheme | N=1 | N=2 | N=4 | e2e N=4 |")
    print("|---|---|---|---|---|---|")
    vals = {}
    for key, cfg, scheme in ROWS:
        cells = []
        for n in (1, 2, 4):
            r = load(d, f"{key}_n{n}")
            vals[(key, n)] = r["value"] if r else None
            cells.append(f"{r['value']:.1f}" if r else "-")
        r4 = load(d, f"{key}_n4")
        cells.append(f"{r4['e2e']['value']:.1f}" if r4 else "-")
        print(f"| {cfg} | {scheme} | " + " | ".join(cells) + " |")
    print()
    print("Speed-ups at N=4:")
    for m in ("c1", "c2", "c3", "c4"):
        for a, b in (("pipe", "sync"), ("pipe_eager", "sync_eager"), ("pipe", "ps"), ("pipe_eager", "ps")):
            x, y = vals.get((f"{m}_{a}", 4)), vals.get((f"{m}_{b}", 4))
            if x and y:
                print(f"- {m.upper()}: {a} / {b} = {x / y:.2f}x")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/matrix")

"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python scripts/launch_summary.py gpurun_out/launches_TAG.csv [window_index] > profiles/TAG_launches_summary.txt

The bench under --profile-mode runs 1 warm-up window + 1 timed window (+ one profiled pass): the
launches are split into windows at each k_tr_init (a window starts with its transcript), and the
summary covers the chosen window (default: the second one).
"""
import csv
import sys
from collections import OrderedDict


def main(path, widx=1):
    rows = []
    with open(path) as f:
        lines = [l for l in f if not l.startswith("==")]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = r.get("Metric Unit", "ns")
        v = float(r["Metric Value"].replace(",", ""))
        us = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v if unit in ("us", "usecond") else v / 1e3
        rows.append((r["Kernel Name"].split("(")[0], us))
    windows, cur = [], []
    for name, us in rows:
        if name.endswith("k_tr_init") and cur:
            windows.append(cur)
            cur = []
        cur.append((name, us))
    if cur:
        windows.append(cur)
    w = windows[min(widx, len(windows) - 1)]
    agg = OrderedDict()
    for name, us in w:
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + us)
    total = sum(t for _, t in agg.values())
    print(f"ncu --metrics gpu__time_duration.sum --clock-control none, one C4 window (window {widx} of {len(windows)};"
          " cold-cache, serialised launches)")
    print(f"launches per window: {len(w)}; total device time {total / 1e3:.3f} ms")
    print(f"{'kernel':44s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'avg_us':>9s}")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:44]:44s} {n:8d} {t / 1e3:9.3f} {100 * t / total:5.1f}% {t / n:9.1f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)

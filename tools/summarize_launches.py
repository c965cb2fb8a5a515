"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel.

    python tools/summarize_launches.py gpurun_out/launches_c3.csv [--md] [--solve-only]
Groups by the demangled kernel name (template arguments kept, namespaces stripped) and grid size,
prints count, total and mean µs, and the share of the total device time.
"""
import csv
import io
import re
import sys
from collections import defaultdict


def load(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    return list(csv.DictReader(io.StringIO("".join(lines))))


def short(name: str) -> str:
    name = re.sub(r"\(.*\)$", "", name)
    name = name.replace("void ", "").replace("amgb::dev::", "").replace("at::native::", "")
    return name[:80]


def main():
    path = sys.argv[1]
    rows = [r for r in load(path) if r["Metric Name"] == "gpu__time_duration.sum"]
    if "--solve-only" in sys.argv:
        # drop the setup-time autotuning launches: a solve starts with the ‖F‖² k_dot
        first = next(i for i, r in enumerate(rows) if "k_dot" in r["Kernel Name"])
        rows = rows[first:]
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        ns = float(r["Metric Value"].replace(",", ""))
        key = (short(r["Kernel Name"]), r["Grid Size"])
        agg[key][0] += 1
        agg[key][1] += ns
        total += ns
    md = "--md" in sys.argv
    if md:
        print("| kernel | grid | launches | total ms | mean µs | share |")
        print("|---|---|---|---|---|---|")
    for (k, g), (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        if md:
            print(f"| `{k}` | {g} | {c} | {ns / 1e6:.3f} | {ns / c / 1e3:.1f} | {100 * ns / total:.1f}% |")
        else:
            print(f"{100 * ns / total:6.2f}%  {ns / 1e6:9.3f} ms  {c:5d}x  {ns / c / 1e3:9.1f} us  {g:>14}  {k}")
    print(f"total {total / 1e6:.3f} ms over {len(rows)} launches")


if __name__ == "__main__":
    main()

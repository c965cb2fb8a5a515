"""Per-kernel DRAM rows from one ncu pass over a solve:

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
l1tex__throughput.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,\
launch__registers_per_thread,launch__grid_size --clock-control none --nvtx --nvtx-include "solve/" --csv \
        --log-file K.csv python tools/profile_solve.py --config C3 --warm 1 --solves 1
    python tools/ncu_kernels.py K.csv [--md out.md] [--peak 6532.9]

Groups launches by kernel (template arguments kept) and grid, and prints per group: launches, mean µs,
DRAM MB per launch (read + write), achieved DRAM GB/s and its fraction of the measured copy peak, L1
throughput and achieved occupancy.  ncu serialises launches and runs them cold (no L2 carry-over
between kernels), so these are per-kernel DRAM figures, not the in-step shares.
"""
import csv
import io
import re
import sys
from collections import defaultdict

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1.0,
        "second": 1.0, "%": 1.0, "": 1.0, "register/thread": 1.0}


def short(name: str) -> str:
    name = re.sub(r"\(.*\)$", "", name).replace("void ", "").replace("amgb::dev::", "").replace("amgb::", "")
    return name


def main():
    path = sys.argv[1]
    md = sys.argv[sys.argv.index("--md") + 1] if "--md" in sys.argv else None
    peak = float(sys.argv[sys.argv.index("--peak") + 1]) if "--peak" in sys.argv else 6532.9
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    per = defaultdict(dict)  # (launch id) -> metrics
    names = {}
    for r in rows:
        lid = (r["ID"], r.get("Kernel Name", ""))
        v = r["Metric Value"].replace(",", "")
        try:
            val = float(v) * UNIT.get(r.get("Metric Unit", ""), 1.0)
        except ValueError:
            continue
        per[lid][r["Metric Name"]] = val
        names[lid] = (short(r["Kernel Name"]), r.get("Grid Size", ""))
    groups = defaultdict(list)
    for lid, m in per.items():
        groups[names[lid]].append(m)
    total = sum(m.get("gpu__time_duration.sum", 0.0) for ms in groups.values() for m in ms)
    out = []
    for (k, grid), ms in groups.items():
        n = len(ms)
        t = sum(m.get("gpu__time_duration.sum", 0.0) for m in ms) / n
        b = sum(m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0) for m in ms) / n
        l1 = sum(m.get("l1tex__throughput.avg.pct_of_peak_sustained_active", 0.0) for m in ms) / n
        occ = sum(m.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0.0) for m in ms) / n
        regs = ms[0].get("launch__registers_per_thread", 0)
        gbs = b / t / 1e9 if t > 0 else 0.0
        out.append(dict(kernel=k, grid=grid, launches=n, us=t * 1e6, share=n * t / total if total else 0.0,
                        dram_mb=b / 1e6, gbs=gbs, frac=gbs / peak, l1=l1, occ=occ, regs=regs))
    out.sort(key=lambda d: -d["share"])
    hdr = "| kernel | grid | launches | share | µs/launch | DRAM MB/launch | DRAM GB/s | frac of peak | L1 % | occupancy % | regs |"
    lines = [hdr, "|" + "---|" * 11]
    for d in out:
        lines.append(f"| `{d['kernel']}` | {d['grid']} | {d['launches']} | {100 * d['share']:.1f} % | {d['us']:.1f} | "
                     f"{d['dram_mb']:.1f} | {d['gbs']:.0f} | {d['frac']:.3f} | {d['l1']:.1f} | {d['occ']:.1f} | {d['regs']:.0f} |")
    text = "\n".join(lines)
    print(text)
    if md:
        with open(md, "w") as f:
            f.write(text + "\n")


if __name__ == "__main__":
    main()

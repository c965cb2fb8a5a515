"""Summarise an ncu --set full capture of the level-0 Chebyshev step (tools/profile_solve.py under ncu)
into profiles/ncu_dominant.json (read by bench.py for roofline.traffic) and a markdown table.

    python tools/ncu_dominant.py gpurun_out/prof.ncu-rep C3 profiles/r01/ncu_c3_cheb_l0.md
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 LSU data-pipe wavefronts %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "of which shared memory %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared-load bank conflicts"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]
UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}


def kernel_key(name: str) -> str:
    """'void k_csr2<8, 6, EpiCheb<0>, ColsD16V16>(...)' -> 'k_csr2<8,6,ColsD16V16>'."""
    m = re.search(r"(k_csr2|k_csr4t)<(\d+), (\d+), [^,]+?(?:<[^>]*>)?, (Cols\w+)>", name)
    if m:
        return f"{m.group(1)}<{m.group(2)},{m.group(3)},{m.group(4)}>"
    m = re.search(r"k_sellviw<(\d+), [\w:]+(?:<[^>]*>)?, (\d+), ", name)  # windowed: 'k_sellviw<U,NBUF>'
    if m:
        return f"k_sellviw<{m.group(1)},{m.group(2)}>"
    m = re.search(r"k_sellvi<(\d+), ", name)  # 'void k_sellvi<2, EpiCheb<0>>(...)' -> 'k_sellvi<2>'
    return f"k_sellvi<{m.group(1)}>" if m else name


def main():
    rep, cfg, md = sys.argv[1], sys.argv[2], sys.argv[3]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    launches = []
    for r in data:
        d = {"kernel": r[col["Kernel Name"]]}
        for m, _ in METRICS:
            if m in col:
                v = r[col[m]].replace(",", "")
                try:
                    d[m] = float(v) * UNIT.get(units[col[m]], 1.0)
                except ValueError:
                    d[m] = v
        launches.append(d)
    main_l = launches[-1]
    key = kernel_key(main_l["kernel"])
    dram = sum(l["dram__bytes_read.sum"] + l["dram__bytes_write.sum"] for l in launches) / len(launches)
    # C3 (the bench default) keeps the historical file name; other workloads get their own file
    name = "ncu_dominant.json" if cfg == "C3" else f"ncu_dominant_{cfg}.json"
    with open(os.path.join(ROOT, "profiles", name), "w") as f:
        json.dump({"workload": cfg, "kernel_key": key, "kernel": main_l["kernel"], "launches": len(launches),
                   "dram_bytes_per_launch": dram, "source": os.path.basename(rep)}, f, indent=1)
    with open(md, "w") as f:
        f.write(f"# ncu --set full: level-0 fused Chebyshev step, {cfg}\n\n")
        f.write(f"Kernel `{main_l['kernel'][:120]}`; {len(launches)} launches captured "
                f"(`{os.path.basename(rep)}`, --clock-control none).\n\n")
        f.write("| metric | " + " | ".join(f"launch {i}" for i in range(len(launches))) + " |\n")
        f.write("|---|" + "---|" * len(launches) + "\n")
        for m, label in METRICS:
            vals = []
            for l in launches:
                v = l.get(m, "")
                if isinstance(v, float):
                    v = (f"{v / 1e9:.4f} GB" if "bytes" in m else f"{v:.3f} GHz" if "per_second" in m
                         else f"{v:.1f}")
                vals.append(str(v))
            f.write(f"| {label} (`{m}`) | " + " | ".join(vals) + " |\n")
        f.write(f"\nDRAM traffic per launch (read + write): {dram / 1e9:.4f} GB.\n")
        # warp stall breakdown (PC sampling) of the last launch
        r = data[-1]
        st = [(h[len("smsp__pcsamp_warps_issue_stalled_"):], r[i]) for h, i in col.items()
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
        st = [(k, float(v.replace(",", ""))) for k, v in st if v not in ("", "n/a")]
        tot = sum(v for _, v in st) or 1.0
        f.write("\nWarp stall reasons (PC sampling, last launch): " +
                ", ".join(f"{k} {100 * v / tot:.1f} %" for k, v in sorted(st, key=lambda kv: -kv[1])[:6]) + ".\n")
    print(key, dram)


if __name__ == "__main__":
    main()

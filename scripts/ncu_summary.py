"""Summarise ncu outputs for profiles/ (run here, no GPU needed).

    python scripts/ncu_summary.py launches <launches.csv> > profiles/rNN_launches.md
    python scripts/ncu_summary.py full <prof.ncu-rep> > profiles/rNN_full.md
"""
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, per = None, {}
    order = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            key = (int(d["ID"]), d["Kernel Name"].split("(")[0])
            if key not in per:
                per[key] = {}
                order.append(key)
            v = float(d["Metric Value"].replace(",", ""))
            unit = d["Metric Unit"]
            scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0,
                     "Gbyte": 1e3}.get(unit, 1.0)
            per[key][d["Metric Name"]] = v * scale
    print("| # | kernel | us | DRAM read MB | DRAM write MB | DRAM GB/s |")
    print("|---|---|---|---|---|---|")
    for key in order:
        m = per[key]
        t = m.get("gpu__time_duration.sum", 0.0)
        rd = m.get("dram__bytes_read.sum", float("nan"))
        wr = m.get("dram__bytes_write.sum", float("nan"))
        gbs = (rd + wr) / t * 1e3 if t else float("nan")
        print(f"| {key[0]} | {key[1]} | {t:.1f} | {rd:.1f} | {wr:.1f} | {gbs:.0f} |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    cols = {name: hdr.index(name) for name, _ in FULL_METRICS if name in hdr}
    kn = hdr.index("Kernel Name")
    print("| kernel | " + " | ".join(f"{lab} ({units[cols[n]]})" for n, lab in FULL_METRICS if n in cols) + " |")
    print("|---|" + "---|" * len(cols))
    for r in rows[2:]:
        vals = " | ".join(r[cols[n]] for n, _ in FULL_METRICS if n in cols)
        print(f"| {r[kn].split('(')[0]} | {vals} |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])

"""Summarise `ncu --page details --csv` + `--page raw` exports (tools/profile_round.sh) into one
table per kernel: duration, DRAM bytes read/written per launch, DRAM % of peak, registers, grid,
achieved warps/SM, SM-active fraction (developer tool)."""
import csv, sys
from pathlib import Path


def details(path):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    iS, iM, iV = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Value")
    return {(r[iS], r[iM]): r[iV] for r in rows[1:] if len(r) > iV}


def raw(path):
    rows = [r for r in csv.reader(open(path)) if r]
    h, units, vals = rows[0], rows[1], rows[-1]
    out = {}
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
        i = h.index(k)
        scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "usecond": 1.0, "us": 1.0,
                 "nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3}.get(units[i], 1.0)
        out[k] = float(vals[i].replace(",", "")) * scale
    return out


d = Path(sys.argv[1])
print(f"{'kernel':20s} {'us':>8s} {'rd MB':>8s} {'wr MB':>8s} {'dram%':>6s} {'regs':>5s} {'grid':>5s} "
      f"{'warps/SM':>8s} {'SMact':>6s}")
for k in sys.argv[2:]:
    de, ra = details(d / f"{k}.csv"), raw(d / f"{k}_raw.csv")
    g = lambda s, m: de.get((s, m), "?")
    act = float(g("GPU Speed Of Light Throughput", "SM Active Cycles").replace(",", ""))
    ela = float(g("GPU Speed Of Light Throughput", "Elapsed Cycles").replace(",", ""))
    print(f"{k:20s} {ra['gpu__time_duration.sum']:8.2f} {ra['dram__bytes_read.sum']:8.2f} "
          f"{ra['dram__bytes_write.sum']:8.2f} {g('GPU Speed Of Light Throughput', 'DRAM Throughput'):>6s} "
          f"{g('Launch Statistics', 'Registers Per Thread'):>5s} {g('Launch Statistics', 'Grid Size'):>5s} "
          f"{g('Occupancy', 'Achieved Active Warps Per SM'):>8s} {act / ela:6.3f}")

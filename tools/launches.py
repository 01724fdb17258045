"""Print an ncu --csv launch list (gpu__time_duration.sum) as a compact table:
  python tools/launches.py gpurun_out/l3.csv [--last N]"""
import csv, sys

def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    out = []
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        if d["Metric Unit"] in ("nsecond", "ns"):
            v /= 1000.0
        elif d["Metric Unit"] in ("msecond", "ms"):
            v *= 1000.0
        out.append((int(d["ID"]), d["Kernel Name"], d["Grid Size"], d["Block Size"], v))
    return out

if __name__ == "__main__":
    rows = load(sys.argv[1])
    last = int(sys.argv[3]) if len(sys.argv) > 3 else len(rows)
    for i, name, g, b, us in rows[-last:]:
        print(f"{i:4d} {us:10.2f} us  grid {g:>16} block {b:>12}  {name[:100]}")

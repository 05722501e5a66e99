"""Per-launch table from an ncu --csv metrics log (development aid).
python scripts/ncu_perlaunch.py LOG.csv [kernel-regex]"""
import csv
import re
import sys
from collections import OrderedDict

rows = OrderedDict()
with open(sys.argv[1]) as fh:
    lines = [l for l in fh if l.startswith('"')]
for r in csv.DictReader(lines):
    k = (int(r["ID"]), r["Kernel Name"].split("(")[0].replace("<unnamed>::", ""))
    v = r["Metric Value"].replace(",", "")
    unit = r["Metric Unit"]
    x = float(v)
    if unit == "Gbyte": x *= 1e9
    elif unit == "Mbyte": x *= 1e6
    elif unit == "Kbyte": x *= 1e3
    elif unit in ("msecond", "ms"): x *= 1e3
    elif unit in ("nsecond", "ns"): x *= 1e-3
    rows.setdefault(k, {})[r["Metric Name"]] = x
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
tot = {}
for (i, name), m in rows.items():
    t = m.get("gpu__time_duration.sum", 0.0)
    b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    a = tot.setdefault(name, [0, 0.0, 0.0])
    a[0] += 1; a[1] += t; a[2] += b
    if pat and pat.search(name):
        print(f"{i:5d} {name:28s} {t:9.1f} us {b / 1e9:8.3f} GB {b / max(t, 1e-9) / 1e3:7.0f} GB/s "
              f"warps {m.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):5.1f}%")
print("--- totals")
for name, (n, t, b) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"{name:28s} n={n:5d} {t / 1e3:9.2f} ms {b / 1e9:9.2f} GB {b / max(t, 1e-9) / 1e3:7.0f} GB/s")

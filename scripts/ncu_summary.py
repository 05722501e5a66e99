"""Summarise ncu CSV logs (run here, on the CPU box).

  python scripts/ncu_summary.py launches <csv>   per-kernel launch count / time / share
  python scripts/ncu_summary.py traffic <csv>    per-kernel dram bytes per launch
"""
import collections, csv, json, re, sys


def rows(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    r = list(csv.reader(lines))
    return r[0], r[1:]


def kname(s):
    m = re.search(r"(k_[a-z_]+|cub::[A-Za-z]+|[A-Za-z_]+Kernel[A-Za-z_]*)", s)
    return m.group(1) if m else s[:40]


def to_unit(v, unit):
    v = float(v.replace(",", ""))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
             "second": 1e6, "s": 1e6, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
             "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return v * scale.get(unit, 1.0)


def main():
    kind, path = sys.argv[1], sys.argv[2]
    h, data = rows(path)
    ki, mi, vi, ui, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.defaultdict(set)
    for r in data:
        k = kname(r[ki])
        per[k][r[mi]] += to_unit(r[vi], r[ui])
        cnt[k].add(r[ii])
    if kind == "launches":
        tot = sum(d["gpu__time_duration.sum"] for d in per.values())
        out = []
        for k, d in sorted(per.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
            t = d["gpu__time_duration.sum"]
            out.append({"kernel": k, "launches": len(cnt[k]), "total_us": round(t, 1), "share": round(t / tot, 4)})
        print(json.dumps({"total_us": round(tot, 1), "kernels": out}, indent=1))
    else:
        out = {}
        for k, d in per.items():
            n = len(cnt[k])
            b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
            out[k] = {"launches": n, "dram_bytes": b, "dram_bytes_per_launch": b / n,
                      "time_us": d.get("gpu__time_duration.sum", 0)}
        print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

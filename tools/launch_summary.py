"""Summarise an ncu --csv launch list: per kernel name, count / total / avg time
and DRAM bytes.  Usage: python tools/launch_summary.py launches.csv [--last-run]"""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        rec = per.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0].replace("void ", ""),
                                       "grid": d["Grid Size"]})
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3,
                 "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        rec[d["Metric Name"]] = v * scale
    return list(per.values())


def main():
    recs = load(sys.argv[1])
    if "--last-half" in sys.argv:
        recs = recs[len(recs) // 2:]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for r in recs:
        a = agg[r["name"]]
        a[0] += 1
        a[1] += r.get("gpu__time_duration.sum", 0.0)
        a[2] += r.get("dram__bytes_read.sum", 0.0) + r.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{'kernel':58s} {'n':>5s} {'total_us':>10s} {'avg_us':>8s} {'share':>6s} {'dram_GB/s':>10s}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:58]:58s} {n:5d} {t:10.1f} {t / n:8.2f} {t / tot:6.3f} {b / (t * 1e-6) / 1e9 if t else 0:10.1f}")
    print(f"total kernel time {tot:.1f} us over {sum(a[0] for a in agg.values())} launches")


if __name__ == "__main__":
    main()

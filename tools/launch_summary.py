"""Summarise an ncu --csv launch list: per-kernel count, mean time, share, DRAM bytes."""
import csv
import sys
from collections import OrderedDict


def main(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    I = {h: i for i, h in enumerate(hdr)}
    per = OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        key = (r[I["ID"]], r[I["Kernel Name"]])
        per.setdefault(key, {})[r[I["Metric Name"]]] = float(r[I["Metric Value"]].replace(",", ""))
    agg = OrderedDict()
    for (kid, name), m in per.items():
        short = name.split("(")[0].replace("void ", "")[:70]
        a = agg.setdefault(short, {"n": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0})
        a["n"] += 1
        a["ns"] += m.get("gpu__time_duration.sum", 0)
        a["rd"] += m.get("dram__bytes_read.sum", 0)
        a["wr"] += m.get("dram__bytes_write.sum", 0)
    tot = sum(a["ns"] for a in agg.values())
    print(f"{'kernel':72s} {'n':>4s} {'mean ms':>9s} {'share':>6s} {'rd GB/l':>8s} {'wr GB/l':>8s}")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        n = a["n"]
        print(f"{k:72s} {n:4d} {a['ns'] / n / 1e6:9.3f} {a['ns'] / tot:6.1%} {a['rd'] / n / 1e9:8.3f} {a['wr'] / n / 1e9:8.3f}")
    print(f"total {tot / 1e6:.3f} ms over {sum(a['n'] for a in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])

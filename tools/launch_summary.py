"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes])
into per-kernel shares: python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
         "byte": 1.0, "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def load(path):
    hdr = None
    per = collections.OrderedDict()
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = d["ID"]
        e = per.setdefault(key, {"name": d["Kernel Name"]})
        e[d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
    return list(per.values())


def main(path):
    launches = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for e in launches:
        n = e["name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        a = agg[n]
        a[0] += 1
        a[1] += e.get("gpu__time_duration.sum", 0.0)
        a[2] += e.get("dram__bytes_read.sum", 0.0) + e.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | share | avg us | avg DRAM MB | DRAM GB/s |")
    print("|---|---|---|---|---|---|")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = f"{b / t / 1e3:.0f}" if b else "-"
        mb = f"{b / n / 1e6:.2f}" if b else "-"
        print(f"| `{k}` | {n} | {100 * t / tot:.1f}% | {t / n:.2f} | {mb} | {gbs} |")
    print(f"\ntotal {len(launches)} launches, {tot / 1e3:.2f} ms (ncu: cold cache, serialised)")


if __name__ == "__main__":
    main(sys.argv[1])

"""Per-kernel breakdown of the last DiT step in an ncu launch list."""
import collections
import csv
import sys


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
hdr = None
per = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    e = per.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0][-42:], "grid": d["Grid Size"]})
    e[d["Metric Name"]] = f(d["Metric Value"])
L = list(per.values())
idx = [i for i, e in enumerate(L) if "dit_noise" in e["name"]][-1]
agg = collections.OrderedDict()
for e in L[idx:]:
    a = agg.setdefault((e["name"], e["grid"]), [0, 0.0])
    a[0] += 1
    a[1] += e.get("gpu__time_duration.sum", 0) / 1e3
tot = sum(a[1] for a in agg.values())
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| `{k[0]}` | {k[1]} | {a[0]} | {a[1]:.1f} | {a[1] / a[0]:.2f} |")
print(f"total {tot:.1f} us (ncu: serialised, cold)")

"""Summarise an ncu --csv launch list: per kernel name, count / mean us / DRAM GB."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
per = collections.defaultdict(dict)
for d in data:
    v = float(d["Metric Value"].replace(",", ""))
    u = d["Metric Unit"]
    scale = {"ns": 1e-3, "us": 1, "usecond": 1, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3,
             "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1}.get(u, 1)
    per[(int(d["ID"]), d["Kernel Name"].split("(")[0][-40:])][d["Metric Name"]] = v * scale
agg = collections.OrderedDict()
for (i, name), m in sorted(per.items()):
    a = agg.setdefault(name, [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0)
    a[2] += m.get("dram__bytes_read.sum", 0)
    a[3] += m.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':42s} {'n':>4s} {'mean_us':>10s} {'share':>6s} {'rdGB':>7s} {'wrGB':>7s} {'TB/s':>6s}")
for name, (n, t, rd, wr) in agg.items():
    print(f"{name:42s} {n:4d} {t / n:10.1f} {t / tot:6.1%} {rd / n:7.3f} {wr / n:7.3f} {(rd + wr) / t * 1e-3 * 1e6 / 1e6:6.2f}")

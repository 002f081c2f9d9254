"""Aggregate an ncu launch list (gpu__time_duration + dram bytes per launch) by kernel name.
usage: python tools/launch_summary.py launches.csv [last_n_launches]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    data.setdefault((int(d["ID"]), d["Kernel Name"]), {})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
items = list(data.items())
if len(sys.argv) > 2:
    items = items[-int(sys.argv[2]):]
scale_t = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
scale_b = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}
agg = collections.OrderedDict()
tot = 0.0
for (i, name), m in items:
    short = name.split("(")[0].replace("void ", "").replace("wl::", "").replace("(anonymous namespace)::", "")
    short = short.split("::")[-1]
    t = m["gpu__time_duration.sum"]
    ms = t[0] * scale_t.get(t[1], 1.0)
    gb = sum(m[k][0] * scale_b.get(m[k][1], 1.0) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in m)
    a = agg.setdefault(short, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += ms
    a[2] += gb
    tot += ms
print(f"{'kernel':32s} {'launches':>8s} {'ms':>10s} {'share':>6s} {'DRAM GB':>9s} {'GB/launch':>9s} {'DRAM GB/s':>9s}")
for k, (n, ms, gb) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:32s} {n:8d} {ms:10.2f} {ms/tot:6.3f} {gb:9.2f} {gb/n:9.3f} {gb/ms*1e3 if ms else 0:9.0f}")
print(f"total {tot:.1f} ms over {len(items)} launches (cold-cache, serialised: compare shares)")

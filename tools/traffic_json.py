"""profiles/ncu_traffic.json from the ncu launch lists of the C4 bench (tools/r2_ncu_final.sh): mean DRAM
read+write bytes per launch of the Z-step SpMM scope (row kernel + isolated-row stream), the dot pass and the
3-output update pass, per storage mode.
usage: python tools/traffic_json.py f64.csv f32.csv git_hash"""
import collections
import csv
import json
import sys


def per_kernel(path, last=600):
    rows = list(csv.reader(open(path)))
    hdr, data = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        d = dict(zip(hdr, r))
        data.setdefault((int(d["ID"]), d["Kernel Name"]), {})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    agg = collections.defaultdict(list)
    for (_, name), m in list(data.items())[-last:]:
        b = sum(m[k][0] * scale[m[k][1]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in m)
        agg[name.split("(")[0]].append(b)
    return {k: sum(v) / len(v) for k, v in agg.items()}


def pick(tab, *subs):
    for k, v in tab.items():
        if all(s in k for s in subs):
            return v
    return None


out = {"_source": "mean DRAM read+write per launch over the last 600 launches (the timed and warm-up steps) of the C4 bench (B=11, k=30, TOAR), "
                  "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
                  "(tools/r2_ncu_final.sh; profiles/r02_launches_bench_c4*.csv); spmv_binned = the Z-step row kernel + "
                  "spmv_iso_kernel of one launch scope",
       "git": sys.argv[3]}
for mode, path, ty, vw in (("f64", sys.argv[1], "double", "4"), ("f32", sys.argv[2], "float", "8")):
    tab = per_kernel(path)   # (the fp32 list also holds create-time double kernels: t' is computed in double)
    row = pick(tab, f"spmv_binned_kernel<4, 0, {vw}, 0, {ty}>")
    iso = pick(tab, f"spmv_iso_kernel<{ty}>") or 0.0
    dots = pick(tab, f"dcgs2_dots_ring<{ty}>")
    upd = pick(tab, f"toar_update_ring<3, {ty}>")
    out[mode] = {"spmv_binned": {"dram_bytes_per_launch": (row or 0.0) + iso},
                 "dcgs2_dots": {"dram_bytes_per_launch": dots},
                 "toar_update": {"dram_bytes_per_launch": upd}}
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))

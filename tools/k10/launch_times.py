"""Per-kernel mean gpu__time_duration from an ncu --csv launch log (stdin)."""
import collections
import csv
import io
import sys

txt = sys.stdin.read().splitlines()
start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
agg = collections.OrderedDict()
for r in csv.DictReader(io.StringIO("\n".join(txt[start:]))):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    us = {"ns": v / 1e3, "us": v, "ms": v * 1e3}[r["Metric Unit"]]
    a = agg.setdefault(r["Kernel Name"].split("(")[0], [0, 0.0])
    a[0] += 1
    a[1] += us
for k, (n, us) in agg.items():
    print(f"{k[:60]:60s} x{n}  mean {us / n:9.1f} us")

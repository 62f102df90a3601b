"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list.
  python tools/launch_summary.py launches.csv [out.json]"""
import collections
import csv
import json
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if len(r) <= iv:
        continue
    v = float(r[iv].replace(",", ""))
    ns = v * {"us": 1e3, "ms": 1e6, "s": 1e9}.get(r[iu], 1.0) if r[iu] != "ns" else v
    k = r[ik].split("(")[0]
    agg[k][0] += 1
    agg[k][1] += ns
tot = sum(v[1] for v in agg.values())
out = {"unit": "ns (gpu__time_duration.sum, cold-cache, serialised)", "total_ns": tot,
       "kernels": {k: {"launches": v[0], "time": v[1], "share_pct": round(100 * v[1] / tot, 2)}
                   for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}}
for k, v in list(out["kernels"].items())[:15]:
    print(f"{v['time'] / 1e6:10.2f} ms {v['launches']:6d} {v['share_pct']:6.2f}%  {k[:70]}")
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)

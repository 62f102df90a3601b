"""Per-launch table of an ncu --metrics ... --csv launch list (kernels >= 0.2 ms or K4).
python tools/launch_table.py launches.csv"""
import csv, sys
from collections import OrderedDict
lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
L = OrderedDict()
for r in rows[1:]:
    L.setdefault((r[0], r[ik].split("(")[0]), {})[r[im]] = r[iv]
tot = {}
for (i, k), m in L.items():
    t = float(m["gpu__time_duration.sum"].replace(",", ""))
    tot[k] = tot.get(k, 0) + t
    if "sim" in k or "lane" in k or t > 200000:
        print(i, k[:45], f"{t/1e6:.2f} ms", *[m.get(x, "") for x in hdr if False],
              *(m.get(x) for x in m if x != "gpu__time_duration.sum"))
print("totals (ms):", {k[-30:]: round(v / 1e6, 2) for k, v in sorted(tot.items(), key=lambda x: -x[1])[:8]})

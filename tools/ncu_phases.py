"""Buckets an ncu source page (per CUDA line) of k_sim into phases.
python tools/ncu_phases.py src.csv"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
f = "?"
buckets = {}
def phase(fname, ln):
    if not fname.endswith("k_cost.cu"):
        return fname.split("/")[-1]
    for name, lo, hi in [("acquire/unrank", 249, 314), ("future_blocks", 198, 247), ("service_bound", 182, 196),
                         ("kth_select", 316, 393), ("A", 445, 505), ("B_fast", 507, 539), ("B_busy", 540, 578),
                         ("B_update", 579, 608), ("C", 610, 648), ("D", 650, 699)]:
        if lo <= ln <= hi:
            return name
    return "other"
ts = te = 0
for r in rows:
    if r and r[0] == "File Path":
        f = r[1]; continue
    if len(r) < 8 or r[2] != "-":
        continue
    try:
        s, e, ln = int(r[4]), int(r[7]), int(r[0])
    except ValueError:
        continue
    p = phase(f, ln)
    b = buckets.setdefault(p, [0, 0])
    b[0] += s; b[1] += e; ts += s; te += e
for p, (s, e) in sorted(buckets.items(), key=lambda x: -x[1][0]):
    print(f"{p:16s} samples {100*s/ts:5.1f}%  inst {100*e/te:5.1f}%")

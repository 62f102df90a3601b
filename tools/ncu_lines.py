"""Per-CUDA-source-line warp-stall samples and executed instructions of one
kernel in an ncu report (ncu --import-source on).  python tools/ncu_lines.py rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
print(rows[1][1] if len(rows) > 1 else "?")
lines, tot_s, tot_e = [], 0, 0
for r in rows[3:]:
    if len(r) < 8 or r[2] != "-":
        continue
    try:
        s, e = int(r[4]), int(r[7])
    except ValueError:
        continue
    tot_s += s
    tot_e += e
    lines.append((s, e, r[0], r[1]))
print(f"samples {tot_s}  instructions {tot_e}")
for s, e, ln, src in sorted(lines, key=lambda x: -x[0])[:top]:
    print(f"{100 * s / max(1, tot_s):5.1f}% samp {100 * e / max(1, tot_e):5.1f}% inst  L{ln:>4} {src.strip()[:90]}")

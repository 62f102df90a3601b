"""Summarises ncu reports / launch lists into profiles/ (JSON, judged artifacts).

  python tools/summarize_ncu.py report.ncu-rep out.json
  python tools/summarize_ncu.py --launches launches.csv out.json
  python tools/summarize_ncu.py --k4 report.ncu-rep out.json "<source>"   (time-weighted K4 issue summary)
"""
import csv
import io
import json
import math
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__cycles_elapsed.avg.per_second"]


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        k = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                k[m] = r[hdr.index(m)] + (" " + units[hdr.index(m)] if units[hdr.index(m)] else "")
        stalls = [(h, r[i]) for i, h in enumerate(hdr)
                  if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued")]
        vals = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v)) for h, v in stalls
                if v.replace(".", "").isdigit()]
        tot = sum(v for _, v in vals) or 1.0
        k["top_stalls_pct"] = {h: round(100 * v / tot, 1) for h, v in sorted(vals, key=lambda x: -x[1])[:6]}
        try:
            rb = float(r[hdr.index("dram__bytes_read.sum")])
            wb = float(r[hdr.index("dram__bytes_write.sum")])
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            k["dram_bytes_per_launch"] = rb * scale.get(units[hdr.index("dram__bytes_read.sum")], 1) + \
                wb * scale.get(units[hdr.index("dram__bytes_write.sum")], 1)
        except Exception:
            pass
        out.append(k)
    return out


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = {}
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    total = sum(v for _, v in agg.values()) or 1.0
    return {"unit": "ns (gpu__time_duration.sum, cold-cache, serialised)",
            "kernels": {k: {"launches": c, "time": t, "share_pct": round(100 * t / total, 2)}
                        for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])}}


def k4_summary(path, source):
    """Issue / warps-active utilisation of the captured K4 launches, weighted by
    duration.  `path` is an .ncu-rep or the per-kernel JSON this tool wrote for
    one; launches whose counters ncu left unset (nan) are skipped and counted."""
    if path.endswith(".json"):
        with open(path) as f:
            ks = json.load(f)
    else:
        ks = report(path)
    tw = iw = ww = 0.0
    skipped = 0
    for k in ks:
        t = float(k["gpu__time_duration.sum"].split()[0].replace(",", ""))
        ia = float(k["smsp__issue_active.avg.pct_of_peak_sustained_active"].split()[0])
        wa = float(k["sm__warps_active.avg.pct_of_peak_sustained_active"].split()[0])
        if not (math.isfinite(ia) and math.isfinite(wa)):
            skipped += 1
            continue
        tw += t
        iw += t * ia
        ww += t * wa
    return {"source": source, "kernels_captured": len(ks), "kernels_without_counters": skipped,
            "issue_active_pct_time_weighted": round(iw / tw, 2) if tw else None,
            "warps_active_pct_time_weighted": round(ww / tw, 2) if tw else None}


if __name__ == "__main__":
    if sys.argv[1] == "--k4":
        res = k4_summary(sys.argv[2], sys.argv[4] if len(sys.argv) > 4 else sys.argv[2])
        dst = sys.argv[3]
    elif sys.argv[1] == "--launches":
        res = launches(sys.argv[2])
        dst = sys.argv[3]
    else:
        res = report(sys.argv[1])
        dst = sys.argv[2]
    json.dump(res, open(dst, "w"), indent=1)
    print(json.dumps(res, indent=1)[:3000])

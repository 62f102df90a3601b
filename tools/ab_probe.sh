#!/bin/bash
# A/B timing of library variants on one config (development):
#   tools/ab_probe.sh C3 "" as16 ...   ("" = the product library)
cfg=$1; shift
for v in "$@"; do
  echo "== variant '${v}'"
  CG_BUILD_VARIANT="$v" timeout 600 python tools/perf_probe.py "$cfg" - 1 3 2>&1 | grep -E "rep=|ms_k4" | \
    python -c "import sys,json
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('   ms_total %.1f ms_k4 %.1f steps %d ovf %s' % (d['ms_total'], d['ms_k4'], d['request_steps'], d.get('plans_overflow')))
    else: print(l)"
done

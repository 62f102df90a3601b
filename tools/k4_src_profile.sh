#!/bin/bash
# ncu source-level capture of one K4 launch of a sweep.
#   tools/k4_src_profile.sh <config> <kernel-regex> <launch-skip> <out-name>
#   e.g. tools/k4_src_profile.sh C3 'k_lane<1, 16>' 1 prof_l16_c3
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:${2:-k_sim}" --launch-skip ${3:-0} --launch-count 1 \
    -o gpurun_out/${4:-prof_k4_src} -f python tools/perf_probe.py ${1:-C2} - 1 1 > gpurun_out/${4:-prof_k4_src}.log 2>&1
tail -2 gpurun_out/${4:-prof_k4_src}.log

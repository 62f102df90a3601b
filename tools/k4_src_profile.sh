#!/bin/bash
# ncu source-level capture of one K4 launch (k_sim) on the C2 sweep.
#   tools/k4_src_profile.sh <launch-skip> <out-name>
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sim --launch-skip ${1:-2} --launch-count 1 \
    -o gpurun_out/${2:-prof_k4_src} -f python tools/perf_probe.py C2 - 1 1 > gpurun_out/${2:-prof_k4_src}.log 2>&1
tail -2 gpurun_out/${2:-prof_k4_src}.log

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"k_lane<.int.[12], .int.8>" --launch-skip 2 -c 2 \
    -o gpurun_out/prof_lane -f python tools/perf_probe.py C2 - 1 1 > gpurun_out/prof_lane.log 2>&1
echo rc=$?; tail -2 gpurun_out/prof_lane.log

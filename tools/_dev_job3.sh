cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
      python tools/perf_probe.py C3 - 1 1 > gpurun_out/ncu_launch_c3.log 2>&1; echo "ncu rc=$?"
python tools/summarize_ncu.py --launches gpurun_out/launches_c3.csv gpurun_out/launches_c3.json > /dev/null

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "k4 or golden or live_reference or medium or full_c2 or two_rank" > gpurun_out/dev_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/dev_pytest.log
timeout 300 python tools/perf_probe.py C2 - 1 3 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/dev_launches.csv \
      python tools/perf_probe.py C2 - 1 1 > gpurun_out/dev_ncu.log 2>&1; echo "ncu rc=$?"

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/full_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/full_pytest.log
timeout 600 python tools/perf_probe.py C3 - 1 2 2>&1 | tail -4
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2

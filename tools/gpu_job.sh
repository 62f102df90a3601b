#!/bin/bash
# One GPU session: parity tests, the benchmark line, ncu launch list and full
# captures of the two graded kernels.  Usage: tools/gpu_job.sh [tests] [bench] [ncu] [dev]
#   dev: the K4 parity subset, a C2 timing and a per-launch table (the edit loop)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
what="${*:-tests bench ncu}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
if [[ $what == *tests* ]]; then
  timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -5 gpurun_out/pytest_gpu.log
fi
if [[ $what == *dev* ]]; then
  timeout 900 python -m pytest tests -x -q -m gpu -k "k4 or golden or live_reference or medium or full_c2 or two_rank" \
      > gpurun_out/dev_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/dev_pytest.log
  timeout 300 python tools/perf_probe.py C2 - 1 3 2>&1 | tail -2
  timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
      --clock-control none --csv --log-file gpurun_out/dev_launches.csv python tools/perf_probe.py C2 - 1 1 > /dev/null 2>&1
  python tools/launch_table.py gpurun_out/dev_launches.csv | tail -1
fi
if [[ $what == *bench* ]]; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  tail -c 3000 gpurun_out/bench.json
fi
if [[ $what == *ncu* ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv \
      python tools/perf_probe.py C2 - 1 > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
  timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_(lane|sim)<" -c 16 \
      -o gpurun_out/prof_k4_c2 -f python tools/perf_probe.py C2 - 1 1 > gpurun_out/ncu_k4.log 2>&1; echo "ncu k4 rc=$?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_route_(tma|hist|tile|aggregate)" -s 1 -c 1 \
      -o gpurun_out/prof_k1_c5 -f python tools/k1_probe.py C5 3 > gpurun_out/ncu_k1.log 2>&1; echo "ncu k1 rc=$?"
fi
if [[ $what == *ncu* ]]; then
  # summarise on the box; full-set reports with source can exceed gpurun's copy-back limit
  python tools/summarize_ncu.py --launches gpurun_out/launches_c2.csv gpurun_out/launches_c2.json > /dev/null
  python tools/summarize_ncu.py gpurun_out/prof_k4_c2.ncu-rep gpurun_out/k4_c2_ncu.json > /dev/null
  python tools/summarize_ncu.py --k4 gpurun_out/prof_k4_c2.ncu-rep gpurun_out/k4_ncu_summary.json \
      "ncu --set full --clock-control none -k regex:k_(lane|sim)< -c 16 python tools/perf_probe.py C2 - 1 1" > /dev/null
  python tools/summarize_ncu.py gpurun_out/prof_k1_c5.ncu-rep gpurun_out/k1_c5_ncu.json > /dev/null
  for f in gpurun_out/*.ncu-rep; do [ $(stat -c %s "$f") -gt 20000000 ] && rm -f "$f"; done
  du -sh gpurun_out
fi

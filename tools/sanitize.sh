#!/bin/bash
# compute-sanitizer passes over a parity subset that launches every engine
# kernel family (K1 forms, K2/K3, K4 k_lane/k_sim incl. deep re-runs, K5-K7,
# ingest/json/simulator/drift), on small inputs.  Summaries -> gpurun_out/sanitize_*.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SEL_MEM='golden or k1_forms_exact or edge_request or dp_class4_vs or quality_forms_bit_exact or p95_chunk or sharded_sweep_matches_golden'
SEL_RACE='sweep_matches_golden or rows_match_golden or k1_forms_exact and plain_odd or edge_request_counts and 301 or dp_class4_vs_live_reference and 40 and 301 or quality_forms_bit_exact and ties'
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  case $tool in
    memcheck) sel="$SEL_MEM"; files="tests/test_gpu_parity.py tests/test_gpu_quality.py tests/test_gpu_multirank.py tests/test_ingest.py tests/test_json_writer.py tests/test_simulator.py tests/test_drift.py";;
    *) sel="$SEL_RACE"; files="tests/test_gpu_parity.py tests/test_gpu_quality.py";;
  esac
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 3000 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 --report-api-errors no \
      python -m pytest $files -q -x -m gpu -k "$sel" -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_$tool.log
  grep -E "ERROR SUMMARY|passed|failed|RACECHECK SUMMARY" gpurun_out/sanitize_$tool.log | tail -3
done

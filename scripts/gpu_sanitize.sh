# compute-sanitizer memcheck / racecheck / synccheck on the C1-sized GPU parity tests
set -x
export PYTHONFAULTHANDLER=1
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider \
    -k "c1_whole_stream and static-0 or test_compact_edge_cases or test_kv_edge_cases or test_paged_edge_cases or (c1_windows and 1) or score_random_geometries and 40 and 0.5" \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo $tool rc=$?
  grep -E "ERROR SUMMARY|passed|failed|error" gpurun_out/sanitize_$tool.log | tail -3
done

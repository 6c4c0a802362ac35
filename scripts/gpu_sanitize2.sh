# compute-sanitizer on the round-1 extension kernels: fused score+compact, temporal patches, MV rasterisation,
# similar histogram, NV12 compaction
export PYTHONFAULTHANDLER=1
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider \
    -k "(score_compact_configs and (C1-3-8 or C2-32-4)) or score_compact_generic or (compact_tp_generic and 2) or mv_rasterize or similar_hist or (compact_nv12 and 0)" \
    > gpurun_out/sanitize2_$tool.log 2>&1
  echo $tool rc=$?
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize2_$tool.log | tail -3
done

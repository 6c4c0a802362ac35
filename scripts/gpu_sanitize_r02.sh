# compute-sanitizer memcheck / racecheck / synccheck on the round-2 kernels: the staged NV12 preprocessing (all its
# launcher paths), the shared-memory rasteriser (shift and division paths), the band-staged planar compaction, the
# chained (PDL) fused score+compact.  Outputs in gpurun_out/san2/.
O=gpurun_out/san2; mkdir -p $O
export PYTHONFAULTHANDLER=1
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider \
    -k "compact_nv12_paths or (compact_nv12 and clip and (geom0 or geom1)) or mv_rasterize or (compact_configs and C2) or pdl" \
    > $O/$tool.log 2>&1
  echo $tool rc=$?
  grep -E "ERROR SUMMARY|passed|failed" $O/$tool.log | tail -3
done

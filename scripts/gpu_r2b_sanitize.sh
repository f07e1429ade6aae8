# compute-sanitizer on the round-2 final code (subtree-aligned tiles, 128-row COLMAX, DMMA index prefetch / batched epilogue)
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do for c in p3d12r bbd dense p3d10; do
  [ "$tool" == "racecheck" ] && [ "$c" == "p3d10" ] && continue
  echo "== $tool $c"; timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py $c 2>&1 | tail -4
done; done > gpurun_out/r2b_sanitizer.txt 2>&1
grep -E "==|ERROR SUMMARY|RACECHECK SUMMARY|relres|rror" gpurun_out/r2b_sanitizer.txt | head -60

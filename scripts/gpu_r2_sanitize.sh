mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do for c in p3d10 bbd dense; do
  echo "== $tool $c"; timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py $c 2>&1 | tail -4
done; done > gpurun_out/r2_sanitizer.txt 2>&1
cat gpurun_out/r2_sanitizer.txt | grep -E "==|ERROR SUMMARY|relres|Error" | head -60

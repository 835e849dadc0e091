O=gpurun_out/r02san
mkdir -p $O
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_smoke.py > $O/san_$tool.log 2>&1
  echo "== $tool"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard" $O/san_$tool.log | tail -3
done

# Final session call: the round script (smoke, parity suite, bench lines, shard timings, ncu) + sanitizers.
bash scripts/gpu_round.sh
O=gpurun_out/round
for t in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_smoke.py > $O/san_$t.log 2>&1
  echo "$t rc=$?"; tail -2 $O/san_$t.log
done

SAN=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python -m pytest tests/test_gpu_append.py tests/test_gpu_scores_codes.py -x -q 2>&1 | tail -2
python scripts/sanitize_smoke.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"; tail -3 gpurun_out/san_plain.log
for tool in memcheck racecheck synccheck; do
timeout 900 $SAN --tool $tool --error-exitcode 9 python scripts/sanitize_smoke.py > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/san_$tool.log
done

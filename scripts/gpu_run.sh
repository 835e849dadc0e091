SAN=/usr/local/cuda/bin/compute-sanitizer
$SAN --tool memcheck --error-exitcode 9 python scripts/sanitize_smoke.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/san_memcheck.log
$SAN --tool racecheck --error-exitcode 9 python scripts/sanitize_smoke.py > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/san_racecheck.log
$SAN --tool synccheck --error-exitcode 9 python scripts/sanitize_smoke.py > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -4 gpurun_out/san_synccheck.log
$SAN --tool initcheck --error-exitcode 9 python scripts/sanitize_smoke.py > gpurun_out/san_initcheck.log 2>&1; echo "initcheck rc=$?"; tail -4 gpurun_out/san_initcheck.log

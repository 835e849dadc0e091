set -x
python scripts/diag_rt.py 1024 2>&1 | tail -12
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; tail -8 gpurun_out/pytest_all.log
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_fused.log 2>&1; tail -1 gpurun_out/bench_fused.log | grep -o '"ms_per_step.*"roofline"'

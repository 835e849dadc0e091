timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "host" > gpurun_out/pytest_host.log 2>&1; tail -4 gpurun_out/pytest_host.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_e2e.log 2>&1; tail -1 gpurun_out/bench_e2e.log | grep -o '"e2e".*"gpu_launches"'; grep -i "error\|Trace" gpurun_out/bench_e2e.log | head

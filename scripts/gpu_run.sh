python scripts/diag_rt.py 1024 2>&1 | tail -4
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "roundtrip or tc or config" > gpurun_out/pytest_rt.log 2>&1; tail -4 gpurun_out/pytest_rt.log
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_fused.log 2>&1; tail -1 gpurun_out/bench_fused.log | grep -o '"passes.*"roofline"'
ncu --set full --import-source on --clock-control none -k regex:attn_tc_kernel -s 1 -c 1 -o gpurun_out/prof_rt4 python bench.py --config C4 --steps 1 --warmup 3 --no-e2e --no-cpu --no-pass-events > gpurun_out/ncu_rt4.log 2>&1

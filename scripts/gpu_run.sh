set -x
nvidia-smi -L
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -30 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench1.log 2>&1; tail -5 gpurun_out/bench1.log

set -x
nvidia-smi -L
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "tc or scores" > gpurun_out/pytest_tc.log 2>&1; tail -30 gpurun_out/pytest_tc.log
timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench2.log 2>&1; tail -5 gpurun_out/bench2.log

O=gpurun_out/verify
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 400 $O/bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2>> $O/bench.err; tail -c 300 $O/bench_ref.json

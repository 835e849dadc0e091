O=gpurun_out/c2b
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py -q -x > $O/pytest_step.txt 2>&1; tail -3 $O/pytest_step.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "roundtrip or balanced" > $O/pytest_rt.txt 2>&1; tail -2 $O/pytest_rt.txt
for i in 1 2; do
timeout 120 python bench.py --config C2 --pipeline step --steps 100 --no-e2e --no-cpu > $O/bench_C2_step.json 2>&1
timeout 120 python bench.py --config C2 --pipeline step --graph --steps 100 --no-e2e --no-cpu > $O/bench_C2_step_graph.json 2>&1
for f in $O/bench_C2_step.json $O/bench_C2_step_graph.json; do python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', d['ms_per_step'], d['ms_min'], d['ms_back_to_back'], d['gpu_launches'])"; done
done
B="python bench.py --config C2 --pipeline step --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_step.csv $B > /dev/null 2>&1
python scripts/ncu_summary.py --launches $O/launches_step.csv

O=gpurun_out/c2
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py -q -x -k "rt64" > $O/pytest_rt64.txt 2>&1; tail -2 $O/pytest_rt64.txt
B="python bench.py --config C2 --pipeline step --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_step.csv $B > /dev/null 2>&1
B="python bench.py --config C2 --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_fused.csv $B > /dev/null 2>&1
python scripts/ncu_summary.py --launches $O/launches_step.csv
python scripts/ncu_summary.py --launches $O/launches_fused.csv

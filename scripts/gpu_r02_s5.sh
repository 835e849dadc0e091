# Round-2 verification run: GPU tests, bench lines, ncu launch list + --set full of the top kernels.
O=gpurun_out/r02s5
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
timeout 300 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 600 $O/bench_c4.json
timeout 300 python bench.py --pipeline separate --no-e2e > $O/bench_c4_separate.json 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2>&1
timeout 120 python bench.py --config C1 --pipeline step --steps 100 --no-e2e --no-cpu > $O/bench_C1_step.json 2>&1
timeout 120 python bench.py --config C2 --pipeline step --steps 100 --no-e2e --no-cpu > $O/bench_C2_step.json 2>&1
for c in C1 C2 C3; do timeout 200 python bench.py --config $c --steps 50 --no-e2e --no-cpu > $O/bench_$c.json 2>&1; done
timeout 300 python scripts/probes/shard_time.py --steps 50 > $O/shard_time.txt 2>&1
B="python bench.py --config C4 --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches.csv $B > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_tc_kernel|colmax_v4" -s 2 -c 2 -o $O/prof_r02 $B > $O/ncu_full.log 2>&1
tail -2 $O/ncu_full.log

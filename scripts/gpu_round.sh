#!/bin/bash
# One GPU call: smoke, parity suite, default bench line, separate-pipeline bench, per-rank shard timings,
# ncu launch list and a --set full capture of the step's kernels (C4).  Outputs under gpurun_out/round/.
O=gpurun_out/round
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 600 $O/bench.json
timeout 600 python bench.py --pipeline separate --no-e2e --no-cpu > $O/bench_separate.json 2>> $O/bench.err
timeout 300 python scripts/probes/shard_time.py > $O/shard_time.txt 2>&1; cat $O/shard_time.txt
B="python bench.py --config C4 --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches.csv $B > $O/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"colmax_v4|attn_tc_kernel" -s 4 -c 2 -o $O/prof $B > $O/ncu_full.log 2>&1
tail -2 $O/ncu_full.log
ls -la $O

# round-1 official artefacts: bench line, ncu launch list, ncu --set full of the hot kernels
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; tail -1 gpurun_out/bench_r01.json
python bench.py --pipeline separate --no-e2e --no-cpu > gpurun_out/bench_r01_separate.json 2>&1; tail -1 gpurun_out/bench_r01_separate.json | cut -c1-300
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"attn_tc_kernel|colmax_v4" -s 6 -c 2 -o gpurun_out/full_r01 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full_r01.log 2>&1
tail -2 gpurun_out/ncu_full_r01.log

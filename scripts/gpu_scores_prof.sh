O=gpurun_out/sc
mkdir -p $O
timeout 300 python scripts/bench_scores.py > $O/bench.json 2>&1; cat $O/bench.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scores_codes_kernel -s 2 -c 1 -o $O/prof python scripts/bench_scores.py > $O/ncu.log 2>&1
tail -1 $O/ncu.log

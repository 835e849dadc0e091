# Round-2 status run: bench lines C4 (default) and C1-C3, shard timings with the default and forced-balance rules.
O=gpurun_out/r02
mkdir -p $O
timeout 300 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
for c in C1 C2 C3; do timeout 200 python bench.py --config $c --steps 50 --no-e2e --no-cpu > $O/bench_$c.json 2>&1; done
timeout 200 python scripts/probes/shard_time.py --steps 50 > $O/shard_time.txt 2>&1
KVQ_TC_BALANCE=1 timeout 200 python scripts/probes/shard_time.py --steps 50 > $O/shard_time_bal1.txt 2>&1
KVQ_TC_BALANCE=1 timeout 100 python scripts/time_rt.py 8192 1024 > $O/c2_bal1.txt 2>&1
timeout 100 python scripts/time_rt.py 8192 1024 > $O/c2_bal0.txt 2>&1
for f in $O/*.json; do python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',d['ms_per_step'],d.get('ms_min'),d['passes'],d['roofline']['frac'])"; done
cat $O/shard_time.txt $O/shard_time_bal1.txt $O/c2_bal*.txt

O=gpurun_out/abf
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1; tail -1 $O/pytest.txt
: > $O/f.txt
for r in 1 2 3; do for e in KVQ_TC_FASTCONV=0 KVQ_AUTO=1; do
  env $e timeout 300 python scripts/probes/shard_time.py --steps 60 --ns 1,8 | sed "s/^/$e $r /" >> $O/f.txt 2>&1
  env $e timeout 120 python bench.py --config C2 --pipeline step --steps 100 --no-e2e --no-cpu > $O/c.json 2>&1
  python -c "import json;d=json.loads(open('$O/c.json').read().strip().splitlines()[-1]);print('$e C2 step round $r', round(d['ms_per_step']*1e3,2), 'b2b', round(d['ms_back_to_back']*1e3,2))" >> $O/f.txt
  env $e timeout 120 python bench.py --config C2 --steps 100 --no-e2e --no-cpu > $O/c.json 2>&1
  python -c "import json;d=json.loads(open('$O/c.json').read().strip().splitlines()[-1]);print('$e C2 two-call round $r', round(d['ms_per_step']*1e3,2), 'b2b', round(d['ms_back_to_back']*1e3,2))" >> $O/f.txt
done; done
cat $O/f.txt

O=gpurun_out/fc3
mkdir -p $O; : > $O/f.txt
for r in 1 2 3; do for e in KVQ_AUTO=1 KVQ_TC_FASTCONV=1; do
  env $e timeout 300 python scripts/probes/shard_time.py --steps 60 --ns 2,4 | sed "s/^/$e $r /" >> $O/f.txt 2>&1
  env $e timeout 200 python bench.py --config C3 --steps 60 --no-e2e --no-cpu > $O/c.json 2>&1
  python -c "import json;d=json.loads(open('$O/c.json').read().strip().splitlines()[-1]);print('$e C3 round $r', round(d['ms_per_step']*1e3,1), {k:round(v['ms']*1e3,1) for k,v in d['passes'].items()})" >> $O/f.txt
done; done
cat $O/f.txt

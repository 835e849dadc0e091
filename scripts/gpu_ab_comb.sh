O=gpurun_out/abc
mkdir -p $O
cp ab/libkvq_new.so paper_2601_04719_b200/libkvq.so
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1; tail -1 $O/pytest.txt
: > $O/c.txt
for r in 1 2 3; do for v in old new; do cp ab/libkvq_$v.so paper_2601_04719_b200/libkvq.so
  timeout 120 python bench.py --config C2 --pipeline step --steps 100 --no-e2e --no-cpu > $O/c.json 2>&1
  python -c "import json;d=json.loads(open('$O/c.json').read().strip().splitlines()[-1]);print('$v C2 step round $r', round(d['ms_per_step']*1e3,2), 'b2b', round(d['ms_back_to_back']*1e3,2), 'launches', d['gpu_launches'])" >> $O/c.txt
  timeout 200 python bench.py --config C3 --steps 60 --no-e2e --no-cpu > $O/c.json 2>&1
  python -c "import json;d=json.loads(open('$O/c.json').read().strip().splitlines()[-1]);print('$v C3 round $r', round(d['ms_per_step']*1e3,1), 'b2b', round(d['ms_back_to_back']*1e3,1), {k:round(v['ms']*1e3,1) for k,v in d['passes'].items()})" >> $O/c.txt
  timeout 300 python scripts/probes/shard_time.py --steps 60 --ns 1,2,4 | sed "s/^/$v $r /" >> $O/c.txt 2>&1
done; done
cat $O/c.txt
cp ab/libkvq_new.so paper_2601_04719_b200/libkvq.so

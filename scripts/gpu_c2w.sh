O=gpurun_out/c2w
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_step.py tests/test_gpu_parity.py -q -x -k "fused_a1 or large_path or small_and_large or repeatable or balanced or roundtrip" > $O/pytest.txt 2>&1; tail -1 $O/pytest.txt
: > $O/c2.txt
for r in 1 2 3; do for e in KVQ_TC_BALANCE=9 KVQ_TC_BALANCE=0; do
  env $e timeout 120 python bench.py --config C2 --pipeline step --steps 100 --no-e2e --no-cpu > $O/c2.json 2>&1
  python -c "import json;d=json.loads(open('$O/c2.json').read().strip().splitlines()[-1]);print('$e C2 step round $r', round(d['ms_per_step']*1e3,2), 'b2b', round(d['ms_back_to_back']*1e3,2))" >> $O/c2.txt
  env $e timeout 120 python bench.py --config C2 --steps 100 --no-e2e --no-cpu > $O/c2.json 2>&1
  python -c "import json;d=json.loads(open('$O/c2.json').read().strip().splitlines()[-1]);print('$e C2 two-call round $r', round(d['ms_per_step']*1e3,2), 'b2b', round(d['ms_back_to_back']*1e3,2), {k:round(v['ms']*1e3,1) for k,v in d['passes'].items()})" >> $O/c2.txt
done; done
cat $O/c2.txt

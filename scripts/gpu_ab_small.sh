# Full parity suite + smoke on the current build, then an A/B of ab/libkvq_{old,new}.so on C1/C2/C4 bench steps.
O=gpurun_out/absmall
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
: > $O/ab.txt
for r in 1 2; do for v in old new; do cp ab/libkvq_$v.so paper_2601_04719_b200/libkvq.so
  for c in C1 C2 C4; do timeout 300 python bench.py --config $c --no-e2e --no-cpu --steps 100 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(\"$v $c\",round(d[\"ms_per_step\"]*1000,1),\"us scales\",round(d[\"passes\"][\"scales\"][\"ms\"]*1000,1))" >> $O/ab.txt; done; done; done
cp ab/libkvq_new.so paper_2601_04719_b200/libkvq.so
cat $O/ab.txt

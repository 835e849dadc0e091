# PDL A/B: parity suite first, then shard timings with KVQ_PDL=0/1 alternating, then the default bench.
O=gpurun_out/pdl
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
: > $O/ab.txt
for r in 1 2; do for v in 0 1; do echo "== KVQ_PDL=$v round $r" >> $O/ab.txt; KVQ_PDL=$v timeout 300 python scripts/probes/shard_time.py --steps 100 >> $O/ab.txt 2>&1; done; done
cat $O/ab.txt
timeout 900 python bench.py --no-cpu > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json

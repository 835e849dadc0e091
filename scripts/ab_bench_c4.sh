# A/B of prebuilt libkvq.so variants on the default C4 bench line (sustained, 100 steps), alternating.
O=gpurun_out/ab
mkdir -p $O; : > $O/ab_bench.txt
L=paper_2601_04719_b200/libkvq.so
for r in 1 2 3; do
  for v in ${VARIANTS:-old new}; do
    cp ab/libkvq_$v.so $L
    timeout 200 python bench.py --no-e2e --no-cpu ${BENCH_ARGS:-} 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$v', round(d['ms_per_step'],4), round(d['ms_back_to_back'],4), {k:round(v['ms'],4) for k,v in d['passes'].items()}, d['clocks']['sm_mhz'], d['clocks']['reasons'], d['clocks'].get('power_w'))" >> $O/ab_bench.txt
  done
done
cat $O/ab_bench.txt

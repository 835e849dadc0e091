# A/B of prebuilt libkvq variants (ab/libkvq_<v>.so) on the C4 bench line (and C2/C3 with CONFIGS), alternating.
O=gpurun_out/ab
mkdir -p $O; : > $O/ab_bench.txt
L=paper_2601_04719_b200/libkvq.so
for r in 1 2; do
  for v in ${VARIANTS:-old new}; do
    cp ab/libkvq_$v.so $L
    for c in ${CONFIGS:-C4}; do
      timeout 300 python bench.py --config $c --no-e2e --no-cpu --steps 60 > $O/b_$v_$c.json 2>&1
      python -c "import json;d=json.loads(open('$O/b_$v_$c.json').read().strip().splitlines()[-1]);p=d['passes'];print('$v $c round $r', 'step', round(d['ms_per_step'],4), 'b2b', round(d['ms_back_to_back'],4), {k:round(v['ms'],4) for k,v in p.items()}, 'clk', d['clocks']['sm_mhz'], 'W', d['clocks'].get('power_w'))" >> $O/ab_bench.txt 2>&1
    done
  done
done
cat $O/ab_bench.txt

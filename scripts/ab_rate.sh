# A/B of prebuilt libkvq.so files (ab/libkvq_<v>.so) on the per-CTA rate probe and C2/C3/C4 roundtrip timing.
O=gpurun_out/ab
mkdir -p $O; : > $O/ab_rate.txt
L=paper_2601_04719_b200/libkvq.so
for r in 1 2; do
  for v in ${VARIANTS:-old new}; do
    cp ab/libkvq_$v.so $L
    echo "== $v round $r" >> $O/ab_rate.txt
    TILES=${TILES:-16,128,148,1024} KVQ_TC_BALANCE=0 timeout 300 python scripts/probes/cta_rate.py >> $O/ab_rate.txt 2>&1
    timeout 300 python scripts/time_rt.py 8192 1024 >> $O/ab_rate.txt 2>&1
  done
done
cat $O/ab_rate.txt

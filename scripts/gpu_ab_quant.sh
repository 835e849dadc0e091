O=gpurun_out/abq2
mkdir -p $O; : > $O/q.txt
L=paper_2601_04719_b200/libkvq.so
for r in 1 2; do for v in q4 q8 q2 qslab; do cp ab/libkvq_$v.so $L
  echo "== $v $r" >> $O/q.txt; timeout 200 python scripts/time_rt.py >> $O/q.txt 2>&1
done; done
cp ab/libkvq_q4.so $L
cat $O/q.txt

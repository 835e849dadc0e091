# A/B of prebuilt libkvq.so files on the shard-size step timings (scripts/probes/shard_time.py) and C3.
O=gpurun_out/ab
mkdir -p $O; : > $O/ab_shard.txt
L=paper_2601_04719_b200/libkvq.so
for r in 1 2; do
  for v in ${VARIANTS:-old new}; do
    cp ab/libkvq_$v.so $L
    echo "== $v round $r" >> $O/ab_shard.txt
    timeout 300 python scripts/probes/shard_time.py --ns ${NS:-1,2,4,8} --steps 50 >> $O/ab_shard.txt 2>&1
  done
done
cat $O/ab_shard.txt

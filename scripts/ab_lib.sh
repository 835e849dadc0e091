# A/B prebuilt libkvq.so files (ab/libkvq_<v>.so) on the same box, alternating; VARIANTS="old new new:ENV=1".
O=gpurun_out/ab
mkdir -p $O; : > $O/ab.txt
L=paper_2601_04719_b200/libkvq.so
for r in 1 2; do
  for spec in ${VARIANTS:-old new}; do
    v=${spec%%:*}; e=""; [ "$v" != "$spec" ] && e=${spec#*:}
    cp ab/libkvq_$v.so $L
    echo "== $spec round $r" >> $O/ab.txt
    env $e timeout 300 python scripts/probes/shard_time.py --ns ${NS:-1,2,8} --steps 60 >> $O/ab.txt 2>&1
    env $e timeout 300 python scripts/probes/metrics_time.py >> $O/ab.txt 2>&1
  done
done
cat $O/ab.txt

# A/B of environment settings on the shard-size step timings, alternating: ENVS="A=1 B=0" (use NONE for no setting).
O=gpurun_out/ab
mkdir -p $O; : > $O/ab_env.txt
for r in 1 2 3; do
  for e in ${ENVS:-NONE}; do
    echo "== $e round $r" >> $O/ab_env.txt
    if [ "$e" = NONE ]; then timeout 300 python scripts/probes/shard_time.py --ns ${NS:-1,2,4,8} --steps 50 >> $O/ab_env.txt 2>&1;
    else env $e timeout 300 python scripts/probes/shard_time.py --ns ${NS:-1,2,4,8} --steps 50 >> $O/ab_env.txt 2>&1; fi
  done
done
cat $O/ab_env.txt

O=gpurun_out/r64
mkdir -p $O
timeout 120 python scripts/quick_rt.py > $O/quick.txt 2>&1; echo "quick rc=$?" >> $O/quick.txt
cat $O/quick.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py -q -x -k "roundtrip or balanced or fused_a1 or large_path or small_and_large or config" > $O/pytest.txt 2>&1; tail -5 $O/pytest.txt
for i in 1 2; do
  echo "== r64 $i" >> $O/ab.txt; TILES=128,256,1024,2048 timeout 300 python scripts/probes/cta_rate.py >> $O/ab.txt 2>&1
  echo "== rt128 $i" >> $O/ab.txt; KVQ_TC_RT128=1 TILES=128,256,1024 timeout 300 python scripts/probes/cta_rate.py >> $O/ab.txt 2>&1
done
cat $O/ab.txt
timeout 300 python bench.py --no-e2e --no-cpu > $O/bench_c4.json 2>&1; tail -c 1500 $O/bench_c4.json

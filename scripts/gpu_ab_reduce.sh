O=gpurun_out/abr
mkdir -p $O
cp ab/libkvq_new.so paper_2601_04719_b200/libkvq.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py -q -x -k "roundtrip or balanced or config or large_path or c1" > $O/pytest.txt 2>&1; tail -1 $O/pytest.txt
: > $O/shard.txt
for r in 1 2 3; do for v in old new; do cp ab/libkvq_$v.so paper_2601_04719_b200/libkvq.so; echo "== $v $r" >> $O/shard.txt; timeout 300 python scripts/probes/shard_time.py --steps 60 --ns 1,8 >> $O/shard.txt 2>&1; done; done
cat $O/shard.txt
VARIANTS="old new" CONFIGS="C4 C1" bash scripts/gpu_ab_bench.sh
VARIANTS="old new" CONFIGS="C4 C1" bash scripts/gpu_ab_bench.sh | tail -8
cp ab/libkvq_new.so paper_2601_04719_b200/libkvq.so

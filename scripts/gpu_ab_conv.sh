O=gpurun_out/ab
mkdir -p $O
cp ab/libkvq_new.so paper_2601_04719_b200/libkvq.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_step.py -q -x -k "roundtrip or balanced or fused_a1 or large_path or config or structured" > $O/pytest_new.txt 2>&1; tail -2 $O/pytest_new.txt
VARIANTS="old new" TILES=16,128,1024 bash scripts/ab_rate.sh > /dev/null 2>&1; cat $O/ab_rate.txt
VARIANTS="old new" CONFIGS="C4 C3 C2" bash scripts/gpu_ab_bench.sh
cp ab/libkvq_trace.so paper_2601_04719_b200/libkvq.so
TILES=128,1024 timeout 300 python scripts/probes/trace_rt.py > $O/trace_new.txt 2>&1
grep -v "^  *[0-9][0-9] " $O/trace_new.txt
cp ab/libkvq_new.so paper_2601_04719_b200/libkvq.so

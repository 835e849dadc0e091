for h in 0 1 2 3; do
KVQ_TC_HINTS=$h timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_h$h.log 2>&1; echo "hints=$h"; tail -1 gpurun_out/bench_h$h.log | grep -o '"roundtrip": {"ms": [0-9.]*'
KVQ_TC_HINTS=$h ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:attn_tc_kernel -s 1 -c 1 python bench.py --config C4 --steps 1 --warmup 3 --no-e2e --no-cpu --no-pass-events 2>&1 | grep -E "dram__bytes|duration"
done

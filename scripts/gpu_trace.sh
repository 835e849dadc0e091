# Per-CTA timeline (clock64 trace build) and a --set full capture of the roundtrip in the CTA-bound regime
# (16 tiles = 16 CTAs at D = 8192), to attribute the per-K-block chain.
O=gpurun_out/trace
mkdir -p $O
cp paper_2601_04719_b200/libkvq.so /tmp/libkvq_keep.so
KVQ_NVCC_EXTRA="-DKVQ_TRACE" python -m paper_2601_04719_b200.build > $O/build_trace.log 2>&1
TILES=16,148,1024 timeout 300 python scripts/probes/trace_rt.py > $O/trace.txt 2>&1
cp /tmp/libkvq_keep.so paper_2601_04719_b200/libkvq.so
touch paper_2601_04719_b200/libkvq.so
TILES=16,128,1024 timeout 300 python scripts/probes/cta_rate.py > $O/cta_rate.txt 2>&1
TILES=16 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -s 3 -c 1 -o $O/prof_t16 python scripts/probes/cta_rate.py > $O/ncu_t16.log 2>&1
tail -3 $O/ncu_t16.log
cat $O/trace.txt $O/cta_rate.txt

# Per-warp staged-arrival trace + the near-tie repair path's share of the per-CTA time (NODANGER timing build).
O=gpurun_out/trace2
mkdir -p $O
cp paper_2601_04719_b200/libkvq.so /tmp/libkvq_keep.so
KVQ_NVCC_EXTRA="-DKVQ_TRACE" python -m paper_2601_04719_b200.build > $O/build_trace.log 2>&1
TILES=128,1024 timeout 300 python scripts/probes/trace_rt.py > $O/trace.txt 2>&1
KVQ_NVCC_EXTRA="-DKVQ_EXP_NODANGER" python -m paper_2601_04719_b200.build > $O/build_nd.log 2>&1
cp paper_2601_04719_b200/libkvq.so /tmp/libkvq_nd.so
for i in 1 2; do
  cp /tmp/libkvq_nd.so paper_2601_04719_b200/libkvq.so; touch paper_2601_04719_b200/libkvq.so
  echo "== nodanger $i" >> $O/ab.txt; TILES=128,1024 timeout 300 python scripts/probes/cta_rate.py >> $O/ab.txt 2>&1
  cp /tmp/libkvq_keep.so paper_2601_04719_b200/libkvq.so; touch paper_2601_04719_b200/libkvq.so
  echo "== head $i" >> $O/ab.txt; TILES=128,1024 timeout 300 python scripts/probes/cta_rate.py >> $O/ab.txt 2>&1
done
cat $O/trace.txt | grep -v "^  *[0-9][0-9] " ; cat $O/ab.txt

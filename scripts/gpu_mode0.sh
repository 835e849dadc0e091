# MODE 0 (kvq_error_metrics) probe: ring depth 4 vs 5, and one ncu --set full capture at C4.
O=gpurun_out/mode0
mkdir -p $O
python -m paper_2601_04719_b200.build > /dev/null
for i in 1 2; do timeout 300 python scripts/probes/metrics_time.py >> $O/kst4.txt 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_tc_kernel" -s 1 -c 1 -o $O/prof_mode0 python scripts/probes/metrics_time.py > $O/ncu.log 2>&1
KVQ_NVCC_EXTRA=-DKVQ_TC_KST01=5 python -c "from paper_2601_04719_b200 import build as b; b.build(force=True)" > /dev/null
for i in 1 2; do timeout 300 python scripts/probes/metrics_time.py >> $O/kst5.txt 2>&1; done
cat $O/kst4.txt $O/kst5.txt; tail -2 $O/ncu.log

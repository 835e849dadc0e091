O=gpurun_out/ab
mkdir -p $O
VARIANTS="${VARIANTS:-new nomma ast4 k6q3}" TILES=128,1024 bash scripts/ab_rate.sh > /dev/null 2>&1
cp ab/libkvq_trace.so paper_2601_04719_b200/libkvq.so
TILES=1024 timeout 300 python scripts/probes/trace_rt.py > $O/trace_r64.txt 2>&1
cp ab/libkvq_new.so paper_2601_04719_b200/libkvq.so
cat $O/ab_rate.txt; grep -v "^  *[0-9][0-9] " $O/trace_r64.txt

timeout 600 python scripts/bench_append.py > gpurun_out/bench_append.json 2> gpurun_out/bench_append.err; tail -3 gpurun_out/bench_append.err
python -c "
import json
for r in json.load(open('gpurun_out/bench_append.json')): print(r)
"

for f in int4 int2; do timeout 300 python bench.py --format $f --steps 50 --warmup 5 > gpurun_out/bench_$f.json 2> gpurun_out/bench_$f.err; tail -2 gpurun_out/bench_$f.err; done
python - <<'PY'
import json
for f in ("int4","int2"):
    d=json.loads(open(f"gpurun_out/bench_{f}.json").read().strip().splitlines()[-1])
    print(f, d["ms_per_step"], {k:(round(v["ms"],3), round(v["frac_hbm"],3)) for k,v in d["passes"].items()})
PY

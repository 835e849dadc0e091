timeout 900 python -m pytest tests/test_gpu_fp8.py -q -x -p no:cacheprovider > gpurun_out/pytest_fp8.log 2>&1; tail -2 gpurun_out/pytest_fp8.log
timeout 300 python bench.py --format e4m3 --steps 20 --warmup 3 --no-cpu 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], {k:(round(x['ms'],4), round(x['GBps'])) for k,x in d['passes'].items()}, d['fidelity'])"

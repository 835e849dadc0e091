timeout 600 python -m pytest tests -m gpu -q -x -k "comm" 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/bench_tr1.json 2> gpurun_out/bench_tr1.err; tail -2 gpurun_out/bench_tr1.err
python -c "
import json
d=json.loads(open('gpurun_out/bench_tr1.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['config']['comm'], d['fidelity'], d['e2e']['ms_per_step'] if d['e2e'] else None)
"

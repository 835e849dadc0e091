for v in "0 0" "1 1" "4 2" "5 2"; do set -- $v; KVQ_DEQ_VARIANT=$1 KVQ_Q_VARIANT=$2 timeout 300 python bench.py --pipeline separate --steps 20 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('deq=$1 q=$2', {k:(round(x['ms'],4), round(x['GBps'])) for k,x in d['passes'].items()})"; done
KVQ_DEQ_VARIANT=5 KVQ_Q_VARIANT=2 timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "bit_exact or config_full or roundtrip_host or near_ties or exhaustive" 2>&1 | tail -2

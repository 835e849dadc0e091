#!/bin/bash
# A/B of the headline step (100 steps, sustained) between ab_head/ (a git worktree) and this tree.
s() { python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$1', round(d['ms_per_step'],4), {k:round(v['ms'],4) for k,v in d['passes'].items()}, d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
(cd ab_head && timeout 300 python bench.py --no-e2e --no-cpu 2>/dev/null | s HEAD)
timeout 300 python bench.py --no-e2e --no-cpu 2>/dev/null | s NEW8
KVQ_NVCC_EXTRA=-DKVQ_NCONV_W=16 python -m paper_2601_04719_b200.build > /dev/null 2>&1
timeout 300 python bench.py --no-e2e --no-cpu 2>/dev/null | s NEW16
(cd ab_head && timeout 300 python bench.py --no-e2e --no-cpu 2>/dev/null | s HEAD)
python -m paper_2601_04719_b200.build > /dev/null 2>&1
timeout 300 python bench.py --no-e2e --no-cpu 2>/dev/null | s NEW8

KVQ_NVCC_EXTRA=-DKVQ_TRACE python -m paper_2601_04719_b200.build > /dev/null
python - <<'PY'
import torch, sys
sys.path.insert(0,'.')
from paper_2601_04719_b200 import kvq
import os
T,D,nq=131072,8192,64
K=kvq.kvq_synth_fill(T,D,seed=42); Q=kvq.kvq_synth_fill(nq,D,seed=43); s=kvq.kvq_compute_scales(K)
kvq.kvq_roundtrip(K,s,Q); torch.cuda.synchronize()
PY

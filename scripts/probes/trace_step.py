"""Phase timeline (globaltimer, ns) of CTA 0 of step_small_kernel (libkvq built with -DKVQ_TRACE): start,
end of phase A, after grid sync 1, end of phase B, end of phase C, after grid sync 2, end."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2601_04719_b200 import _lib, kvq  # noqa: E402

T, D, nq = 1024, 128, 64
K = kvq.kvq_synth_fill(T, D, seed=42)
Q = kvq.kvq_synth_fill(nq, D, seed=43)
for _ in range(5):
    kvq.kvq_step(K, Q)
torch.cuda.synchronize()
lib = _lib.load()
lib.kvq_debug_step_trace_read.argtypes = [ctypes.c_void_p]
buf = np.zeros(10, dtype=np.uint64)
assert lib.kvq_debug_step_trace_read(buf.ctypes.data) == 0
t = buf.astype(np.int64)
print("A: Q staged", t[7] - t[0], "K colmax", t[8] - t[7], "atomics", t[1] - t[8])
print("phase ns: A", t[1] - t[0], "sync1", t[2] - t[1], "B", t[3] - t[2], "C", t[4] - t[3], "sync2", t[5] - t[4],
      "D", t[6] - t[5], "total", t[6] - t[0])

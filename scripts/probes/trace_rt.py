"""Timeline of CTA 0 of attn_tc_kernel<2> (libkvq built with -DKVQ_TRACE): clock64 per event and K-block.
Events: 0 producer issues load | 1 conv w4 sees full_k | 2 conv w4 arrived staged | 3 conv w4 got empty_a |
4 conv w4 arrived full_a | 5 conv w11 sees full_k | 6 conv w11 arrived full_a | 7 store sees staged |
8 store freed stage g-1 | 9 MMA sees full_a | 10 MMA committed.
    TILES=16 python scripts/probes/trace_rt.py"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2601_04719_b200 import kvq, _lib  # noqa: E402

D, nq = 8192, 64
for tiles in [int(x) for x in os.environ.get("TILES", "16,148").split(",")]:
    T = tiles * 128
    K = kvq.kvq_synth_fill(T, D, seed=42)
    Q = kvq.kvq_synth_fill(nq, D, seed=43)
    s = kvq.kvq_compute_scales(K)
    for _ in range(3):
        kvq.kvq_roundtrip(K, s, Q)
    torch.cuda.synchronize()
    buf = np.zeros((64, 48), dtype=np.uint64)
    lib = _lib.load()
    lib.kvq_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    assert lib.kvq_debug_trace_read(buf.ctypes.data, buf.nbytes) == 0
    t = buf.astype(np.int64)
    base = t[0, 0]
    print(f"== tiles={tiles}: per-block period (ev0 diff, cycles):", np.diff(t[:, 0])[:16].tolist())
    print("  median period per event:", [int(np.median(np.diff(t[:, e]))) for e in range(11)])
    seq = [14, 1, 11, 12, 13, 2, 3, 4]
    d = [int(np.median(t[:, b] - t[:, a])) for a, b in zip(seq, seq[1:])]
    d.append(int(np.median(t[2:, 14] - t[:-2, 4])))
    print("  converter (first warp of the owning team) median segments 14>1 1>11 11>12 12>13 13>2 2>3 3>4 "
          "4>14(same team's next block):", d)
    print("  last warp of the team: full_k seen (5) - first warp (1):", int(np.median(t[:, 5] - t[:, 1])),
          " full_a arrived (6) - (4):", int(np.median(t[:, 6] - t[:, 4])))
    print("  load issue -> full_k seen (0>1):", int(np.median(t[:, 1] - t[:, 0])), " 4 -> MMA sees full_a (9):",
          int(np.median(t[:, 9] - np.maximum(t[:, 4], t[:, 6]))), " MMA 9>10:", int(np.median(t[:, 10] - t[:, 9])),
          " staged(2) -> store sees (7):", int(np.median(t[:, 7] - t[:, 2])), " 7>8:", int(np.median(t[:, 8] - t[:, 7])))
    w = t[:, 16:24]
    wl = t[:, 32:40]
    ok = (w > 0).all(axis=1)
    spread = (w.max(axis=1) - w.min(axis=1))[ok]
    lspread = (wl.max(axis=1) - wl.min(axis=1))[ok]
    print("  staged arrival spread over the team's 8 warps (cycles): median", int(np.median(spread)), " p90",
          int(np.percentile(spread, 90)), " max", int(spread.max()), "; quantize-done spread: median",
          int(np.median(lspread)), " p90", int(np.percentile(lspread, 90)), " max", int(lspread.max()))
    print("  last staged arrival -> store sees (7):", int(np.median((t[:, 7] - w.max(axis=1))[ok])),
          "; which warp is last (counts):", np.bincount(np.argmax(w[ok], axis=1), minlength=8).tolist())
    print("  per block spread:", spread[:24].tolist())
    ev = [0, 14, 1, 11, 2, 3, 4, 7, 8, 9, 10]
    print("  absolute (cycles from block 64's load issue); events " + " ".join(f"{e:>6d}" for e in ev))
    for g in range(0, 24):
        print(f"  {g+64:5d}  " + " ".join(f"{(t[g, e] - base) if t[g, e] else -1:6d}" for e in ev))

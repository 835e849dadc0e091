"""Exercise every libkvq entry point on small ragged shapes (for compute-sanitizer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_04719_b200 import kvq  # noqa: E402

torch.cuda.set_device(0)
for (T, D, nq) in [(300, 64, 7), (129, 48, 64), (77, 13, 5), (1, 4, 1), (257, 1024, 64), (25600, 512, 64)]:
    # the last shape (200 tiles) runs the tensor-core pass with a split tail (forced): whole waves + pieces
    if T == 25600:
        os.environ["KVQ_TC_BALANCE"] = "1"
    K = kvq.kvq_synth_fill(T, D, seed=42, dist=1)
    Q = kvq.kvq_synth_fill(nq, D, seed=43)
    s = kvq.kvq_compute_scales(K)
    q = kvq.kvq_quantize(K, s)
    kh = kvq.kvq_dequantize(q, s)
    q2, kh2 = kvq.kvq_quantize_dequantize(K, s)
    m = kvq.kvq_error_metrics(K, kh, Q, s)
    q3, kh3, out = kvq.kvq_roundtrip(K, s, Q)
    S = kvq.kvq_attention_scores(Q, K, kh)
    s4, q4, kh4, single = kvq.kvq_quantize_fused(K)
    r = kvq.kvq_roundtrip_host(K.cpu().pin_memory(), Q.cpu().pin_memory())
    torch.cuda.synchronize()
    assert torch.equal(q, q2) and torch.equal(q, q3) and torch.equal(q, q4)
    # NEXT rows: FP8, INT4/INT2 packed, scores from codes (int8 tensor cores, CTA pairs), streaming append
    sf = kvq.kvq_compute_scales_fmt(K, kvq.FMT_E4M3)
    q8, kh8 = kvq.kvq_quantize_e4m3(K, sf, want_khat=True)
    kh8b = kvq.kvq_dequantize_e4m3(q8, sf)
    for bits, fmt in ((4, kvq.FMT_INT4), (2, kvq.FMT_INT2)):
        sb = kvq.kvq_compute_scales_fmt(K, fmt)
        pb, khb = kvq.kvq_quantize_packed(K, sb, bits, want_khat=True)
        khb2 = kvq.kvq_dequantize_packed(pb, sb, D, bits)
        assert torch.equal(khb, khb2)
    if nq <= 64:
        Sc = kvq.kvq_scores_from_codes(Q, q, s)
    # kvq_step: the one-launch small path (cooperative grid barriers) and the two-call path
    os.environ["KVQ_STEP_SMALL"] = "1"
    st_s, st_q, st_kh, st_out = kvq.kvq_step(K, Q)
    os.environ["KVQ_STEP_SMALL"] = "0"
    st_s2, st_q2, st_kh2, st_out2 = kvq.kvq_step(K, Q)
    os.environ.pop("KVQ_STEP_SMALL")
    torch.cuda.synchronize()
    assert torch.equal(st_q, q) and torch.equal(st_q2, q)
    cache = kvq.AppendCache(T + 8, D)
    cache.append(K[: T // 2])
    cache.append(K[T // 2: T // 2 + 1] * 3.0)
    cache.append(K[T // 2 + 1: T])
    torch.cuda.synchronize()
    print(T, D, nq, "ok", m["attn_mean_abs"], single)
    os.environ.pop("KVQ_TC_BALANCE", None)
# peer-memory collectives at world 1 (the exchange kernels, the fused column max + exchange + finalize)
for D in (64, 13, 1024):
    p = kvq.Peer(1, 0, D)
    p.open([p.ipc_handle])
    c = kvq.Comm.from_peer(p)
    K = kvq.kvq_synth_fill(200, D, seed=3, dist=1)
    Q = kvq.kvq_synth_fill(9, D, seed=43)
    s = kvq.kvq_compute_scales(K, comm=c)
    if D % 4 == 0:
        s2 = kvq.kvq_compute_scales_peer(K, p)
        assert torch.equal(s, s2)
    _, kh, out = kvq.kvq_roundtrip(K, s, Q, comm=c)
    m = kvq.kvq_error_metrics(K, kh, Q, s, comm=c)
    torch.cuda.synchronize()
    c.destroy()
    p.destroy()
# balanced tail forced on (tiles split between CTAs, split_combine_kernel), tensor-core metrics and roundtrip
os.environ["KVQ_TC_BALANCE"] = "1"
for (T, D, nq) in [(640, 256, 64), (300, 128, 17), (1000, 1024, 33)]:
    K = kvq.kvq_synth_fill(T, D, seed=42, dist=1)
    Q = kvq.kvq_synth_fill(nq, D, seed=43)
    s = kvq.kvq_compute_scales(K)
    q3, kh3, out = kvq.kvq_roundtrip(K, s, Q)
    m = kvq.kvq_error_metrics(K, kh3, Q, s)
    torch.cuda.synchronize()
    print(T, D, nq, "balanced ok", m["attn_mean_abs"])
os.environ.pop("KVQ_TC_BALANCE")

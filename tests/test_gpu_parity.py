"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Codes, scales and K_hat bit-exact; metrics and scores
within the north-star relative tolerance 1e-5 (BASELINE.json north_star)."""
import hashlib
import json
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REL = 1e-5  # north_star: "Error metrics and attention scores must agree within a relative tolerance of 1e-5"
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def kvq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2601_04719_b200 import kvq as k
    k.kvq_device_check()
    return k


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def same_bits(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    assert a.shape == b.shape and a.dtype == b.dtype
    va = a.view(np.uint8 if a.dtype == np.int8 else np.uint32)
    vb = b.view(np.uint8 if b.dtype == np.int8 else np.uint32)
    bad = np.nonzero(va != vb)
    if bad[0].size:
        i = tuple(x[0] for x in bad)
        raise AssertionError(f"{bad[0].size} mismatches; first at {i}: gpu={a[i]!r} oracle={b[i]!r}")


def gpu_roundtrip(kvq, K, fused=False):
    Kd = dev(K)
    s = kvq.kvq_compute_scales(Kd)
    if fused:
        q, kh = kvq.kvq_quantize_dequantize(Kd, s)
    else:
        q = kvq.kvq_quantize(Kd, s)
        kh = kvq.kvq_dequantize(q, s)
    return host(s), host(q), host(kh)


def check_vs_oracle(kvq, orc, K, fused=False):
    s, q, kh = gpu_roundtrip(kvq, K, fused)
    so, qo, kho = orc.roundtrip(K)
    same_bits(s, so)
    same_bits(q, qo)
    same_bits(kh, kho)


# ----------------------------------------------------------------------------- generator
@pytest.mark.parametrize("dist", [0, 1, 2])
def test_device_generator_matches_oracle(kvq, orc, dist):
    for (rows, D, row0) in [(33, 7, 0), (64, 128, 100), (5, 1000, 3)]:
        g = host(kvq.kvq_synth_fill(rows, D, row0=row0, seed=42, dist=dist))
        same_bits(g, orc.fill(rows, D, 42, dist, row0))


# ----------------------------------------------------------------------------- edge battery
EDGE_SHAPES = [(1, 1), (1, 4), (1, 5), (2, 3), (3, 7), (7, 13), (64, 128), (1000, 13), (257, 127),
               (129, 1024), (33, 4096), (5000, 8),
               # row-slab grid: column chunks of 256 float4 with a partial last chunk (D/4 = 257, 300)
               (5, 1028), (33, 1200), (1, 1200)]


@pytest.mark.parametrize("shape", EDGE_SHAPES)
@pytest.mark.parametrize("fused", [False, True])
def test_random_shapes_bit_exact(kvq, orc, shape, fused):
    T, D = shape
    check_vs_oracle(kvq, orc, orc.fill(T, D, 7, 1), fused)


@pytest.mark.parametrize("name", ["zeros", "ones", "alternating", "negzero", "subnormal", "underflow",
                                  "ties", "ongrid", "huge", "mixed_binades"])
def test_structured_inputs_bit_exact(kvq, orc, name):
    """P:538 edge cases (all zeros, all ones, alternating signs) plus the readings' corner cases."""
    rng = np.random.default_rng(3)
    T, D = 96, 20
    if name == "zeros":
        K = np.zeros((T, D), np.float32)
    elif name == "ones":
        K = np.ones((T, D), np.float32)
    elif name == "alternating":
        K = np.where((np.arange(T)[:, None] + np.arange(D)) % 2 == 0, 1.0, -1.0).astype(np.float32) * 0.37
    elif name == "negzero":
        K = np.full((T, D), -0.0, np.float32)
        K[5, 3] = 0.25
    elif name == "subnormal":  # subnormal scales take the exact path; clamp fires (reading Q4)
        K = (rng.uniform(-1, 1, (T, D)) * 2.0 ** -140).astype(np.float32)
        K[0, :] = np.float32(2.0 ** -140)
    elif name == "underflow":  # nonzero columns whose scale underflows to 0 (reading Q5)
        K = (rng.choice([-1, 0, 1], (T, D)) * 2.0 ** -149).astype(np.float32)
    elif name == "ties":  # exact .5 quotients: half-even (reading Q1)
        col = np.array([127, 0.5, 1.5, 2.5, -2.5, -127, 63.5, -0.5, 126.5, -126.5], np.float32) / 128
        K = np.tile(col[:, None], (10, D)).astype(np.float32)
    elif name == "ongrid":
        K = orc.fill(T, D, 5, orc.DIST_ONGRID)
    elif name == "huge":
        K = (rng.uniform(-1, 1, (T, D)) * 3.0e38).astype(np.float32)
    else:
        K = (rng.uniform(-1, 1, (T, D)) * 2.0 ** rng.integers(-60, 60, (T, D))).astype(np.float32)
    for fused in (False, True):
        check_vs_oracle(kvq, orc, K, fused)


def test_misaligned_bases_take_scalar_path(kvq, orc):
    """Any alignment: views at odd element offsets are still bit-exact."""
    T, D = 77, 64
    K = orc.fill(T, D, 9, 1)
    big = torch.zeros(T * D + 3, dtype=torch.float32, device="cuda")
    Kv = big[1:1 + T * D].view(T, D)
    Kv.copy_(dev(K))
    s_buf = torch.zeros(D + 1, dtype=torch.float32, device="cuda")
    s = kvq.kvq_compute_scales(Kv, s_buf[1:])
    qb = torch.zeros(T * D + 3, dtype=torch.int8, device="cuda")
    q = kvq.kvq_quantize(Kv, s, qb[3:].view(T, D))
    khb = torch.zeros(T * D + 2, dtype=torch.float32, device="cuda")
    kh = kvq.kvq_dequantize(q, s, khb[2:].view(T, D))
    so, qo, kho = orc.roundtrip(K)
    same_bits(host(s), so)
    same_bits(host(q), qo)
    same_bits(host(kh), kho)


def test_quantize_with_given_scales_near_ties(kvq, orc):
    """Quantize against arbitrary (not self-computed) scales, dense in near-tie quotients."""
    rng = np.random.default_rng(11)
    D = 64
    s = rng.uniform(1e-3, 10, D).astype(np.float32)
    k = rng.integers(-130, 130, (512, D)).astype(np.float32) + 0.5
    K = (k * s).astype(np.float32)
    K = np.stack([K, np.nextafter(K, np.float32(np.inf)), np.nextafter(K, np.float32(-np.inf))]).reshape(-1, D)
    Kd, sd = dev(K), dev(s)
    same_bits(host(kvq.kvq_quantize(Kd, sd)), orc.quantize(K, s))
    q, kh = kvq.kvq_quantize_dequantize(Kd, sd)
    same_bits(host(q), orc.quantize(K, s))
    same_bits(host(kh), orc.dequantize(orc.quantize(K, s), s))


@pytest.mark.parametrize("scale", [1 / 127, 1.0, 3 * 2.0 ** -10, 0.75 / 127, 2.0 ** -126, 2.0 ** 100 / 127,
                                   1.1754942e-38, 4 * 2.0 ** -149])
def test_quantize_exhaustive_binades(kvq, orc, scale):
    """Every fp32 x with |x/s| in [2^-2, 2^8) (10 binades, both signs) for fixed s:
    all codes, all ties, the clamp region.  Oracle = Listing 3 with Q1/Q2."""
    s = np.float32(scale)
    lo = np.float32(s * 0.25)
    hi = np.float32(s * 256)
    lo_b, hi_b = int(lo.view(np.uint32)), int(hi.view(np.uint32))
    sd = dev(np.array([s], np.float32))
    for c0 in range(lo_b, hi_b, 1 << 25):
        x = np.arange(c0, min(c0 + (1 << 25), hi_b), dtype=np.uint32).view(np.float32)
        x = np.concatenate([x, -x]).reshape(-1, 1)
        got = host(kvq.kvq_quantize(dev(x), sd))
        same_bits(got, orc.quantize(x, np.array([s], np.float32)))


def test_determinism(kvq, orc):
    K = dev(orc.fill(4096, 256, 1))
    outs = []
    for _ in range(3):
        s = kvq.kvq_compute_scales(K)
        q, kh = kvq.kvq_quantize_dequantize(K, s)
        outs.append((host(s).tobytes(), host(q).tobytes(), host(kh).tobytes()))
    assert outs[0] == outs[1] == outs[2]


# ----------------------------------------------------------------------------- metrics + attention
def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.mark.parametrize("T,D,nq", [(1, 1, 1), (1000, 1000, 70), (64, 32, 64), (300, 13, 5), (517, 128, 0)])
def test_metrics_ragged_vs_oracle(kvq, orc, T, D, nq):
    K = orc.fill(T, D, 2, 1)
    s, q, Kh = orc.roundtrip(K)
    Q = orc.fill(nq, D, 43) if nq else None
    m = kvq.kvq_error_metrics(dev(K), dev(Kh), None if Q is None else dev(Q), dev(s))
    ss, mx = orc.recon_errors(K, Kh)
    assert _rel(m["sum_sq"], ss) <= REL or ss == 0
    assert m["max_abs"] == mx  # exact: a max of exact differences
    assert m["theoretical_max"] == orc.theoretical_max(s)
    assert m["n_elems"] == T * D and m["n_scores"] == nq * T
    if nq:
        ref = orc.attention_error(Q, K, Kh)
        assert _rel(m["attn_mean_abs"], ref) <= REL


@pytest.mark.parametrize("with_khat", [False, True])
def test_attention_scores_per_entry(kvq, orc, with_khat):
    T, D, nq = 200, 1000, 67
    K = orc.fill(T, D, 4)
    _, _, Kh = orc.roundtrip(K)
    Q = orc.fill(nq, D, 43)
    S = host(kvq.kvq_attention_scores(dev(Q), dev(K), dev(Kh) if with_khat else None))
    E = (K.astype(np.float64) - Kh.astype(np.float64)) if with_khat else K.astype(np.float64)
    ref = orc.scores(Q, K) - (orc.scores(Q, Kh) if with_khat else 0)
    cond = np.abs(Q.astype(np.float64)) @ np.abs(E).T  # sum_d |Q_id E_td|
    assert np.all(np.abs(S - ref) <= REL * cond + 1e-30)


def test_metrics_identity_is_zero(kvq, orc):
    K = dev(orc.fill(300, 64))
    Q = dev(orc.fill(8, 64, 43))
    m = kvq.kvq_error_metrics(K, K.clone(), Q)
    assert m["l2"] == 0 and m["max_abs"] == 0 and m["attn_mean_abs"] == 0


# ----------------------------------------------------------------------------- configs C1, C2 (full compare)
def gold(cfg):
    with open(os.path.join(GOLD, "survey_appendix.json")) as f:
        return json.load(f)[cfg]


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_config_full_parity(kvq, orc, cfg):
    g = gold(cfg)
    T, D = g["T"], g["D"]
    Kd = kvq.kvq_synth_fill(T, D, seed=42)
    Qd = kvq.kvq_synth_fill(64, D, seed=43)
    s = kvq.kvq_compute_scales(Kd)
    q = kvq.kvq_quantize(Kd, s)
    kh = kvq.kvq_dequantize(q, s)
    m = kvq.kvq_error_metrics(Kd, kh, Qd, s)
    K = orc.fill(T, D)
    so, qo, kho = orc.roundtrip(K)
    same_bits(host(Kd), K)
    same_bits(host(s), so)
    same_bits(host(q), qo)
    same_bits(host(kh), kho)
    assert hashlib.sha256(host(q).tobytes()).hexdigest()[:16] == g["q_sha16"]
    ss, mx = orc.recon_errors(K, kho)
    attn = orc.attention_error(orc.fill(64, D, 43), K, kho)
    assert _rel(m["l2"], math.sqrt(ss)) <= REL and m["max_abs"] == mx
    assert _rel(m["attn_mean_abs"], attn) <= REL
    assert _rel(m["attn_mean_abs"], g["attn_mean_abs"]) <= REL


# ----------------------------------------------------------------------------- configs C3, C4 (hash + samples)
@pytest.mark.parametrize("cfg", ["C3", "C4"])
def test_config_large_parity(kvq, orc, cfg):
    """Full-size outputs hash-equal the SURVEY goldens (independent numpy
    implementation), sampled elements equal the oracle one by one, metrics
    match the goldens, attention matches the oracle on a row block and the
    closed form over all rows."""
    g = gold(cfg)
    T, D = g["T"], g["D"]
    Kd = kvq.kvq_synth_fill(T, D, seed=42)
    Qd = kvq.kvq_synth_fill(64, D, seed=43)
    s = kvq.kvq_compute_scales(Kd)
    q = kvq.kvq_quantize(Kd, s)
    kh = kvq.kvq_dequantize(q, s)
    m = kvq.kvq_error_metrics(Kd, kh, Qd, s)
    sh = host(s)
    assert hashlib.sha256(sh.tobytes()).hexdigest()[:16] == g["scales_sha16"]
    assert hashlib.sha256(host(q).tobytes()).hexdigest()[:16] == g["q_sha16"]
    hk = hashlib.sha256()
    for r0 in range(0, T, 8192):
        hk.update(host(kh[r0:r0 + 8192]).tobytes())
    assert hk.hexdigest()[:16] == g["khat_sha16"]
    assert _rel(m["l2"], g["l2"]) <= REL and m["max_abs"] == g["max_abs"]
    # sampled elements vs the oracle, one by one (scales from the streamed oracle)
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(T, 64, replace=False))
    so = orc.streamed_pipeline(T, D, hashes=False, block_rows=2048)["scales"] if cfg == "C3" else sh
    if cfg == "C3":
        same_bits(sh, so)
    for r in rows:
        Kr = orc.fill(1, D, 42, 0, int(r))
        qo = orc.quantize(Kr, so)
        same_bits(host(q[r:r + 1]), qo)
        same_bits(host(kh[r:r + 1]), orc.dequantize(qo, so))
    # attention: one 64-row block against the oracle, whole matrix against the closed form
    r0 = int(rows[0])
    blk = slice(r0, r0 + 64)
    Kb = orc.fill(64, D, 42, 0, r0)
    Khb = orc.dequantize(orc.quantize(Kb, so), so)
    Qh = orc.fill(64, D, 43)
    mb = kvq.kvq_error_metrics(Kd[blk].contiguous(), kh[blk].contiguous(), Qd)
    assert _rel(mb["attn_mean_abs"], orc.attention_error(Qh, Kb, Khb)) <= REL
    closed = math.sqrt(2 / math.pi) * float(np.mean(sh)) * math.sqrt(D / 12) * math.sqrt(1 / 3)
    assert m["attn_mean_abs"] == pytest.approx(closed, rel=0.01)
    assert abs(m["attn_mean_abs"] - 0.095) < 0.002


# ----------------------------------------------------------------------------- host pipeline + comm
def test_roundtrip_host_matches_device_path(kvq, orc):
    T, D, nq = 3000, 256, 64
    K = orc.fill(T, D, 42)
    Q = orc.fill(nq, D, 43)
    Kh_host = torch.empty((T, D), dtype=torch.float32).pin_memory()
    r = kvq.kvq_roundtrip_host(torch.from_numpy(K).pin_memory(), torch.from_numpy(Q).pin_memory(),
                               K_hat_host=Kh_host)
    so, qo, kho = orc.roundtrip(K)
    same_bits(r["scales"].numpy(), so)
    same_bits(r["Kq"].numpy(), qo)
    same_bits(Kh_host.numpy(), kho)
    ss, mx = orc.recon_errors(K, kho)
    assert _rel(r["metrics"]["sum_sq"], ss) <= REL and r["metrics"]["max_abs"] == mx
    assert _rel(r["metrics"]["attn_mean_abs"], orc.attention_error(Q, K, kho)) <= REL


def test_single_rank_comm_path(kvq, orc):
    """The NCCL exchange path with one rank must not change any result."""
    uid = kvq.kvq_comm_unique_id()
    comm = kvq.Comm(uid, 1, 0)
    try:
        K = orc.fill(700, 96, 42, 1)
        Kd = dev(K)
        s = kvq.kvq_compute_scales(Kd, comm=comm)
        so, qo, kho = orc.roundtrip(K)
        same_bits(host(s), so)
        q, kh = kvq.kvq_quantize_dequantize(Kd, s)
        m = kvq.kvq_error_metrics(Kd, kh, dev(orc.fill(8, 96, 43)), s, comm=comm)
        assert m["max_abs"] == orc.max_abs_error(K, kho)
    finally:
        comm.destroy()


# ----------------------------------------------------------------------------- tensor-core (tcgen05) attention path
TC_CASES = [(1, 4, 1), (128, 32, 64), (129, 36, 64), (1000, 1000, 64), (300, 128, 17), (257, 8192, 64),
            (4096, 1024, 64), (64, 4, 3)]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("T,D,nq", TC_CASES)
def test_tc_metrics_vs_oracle(kvq, orc, T, D, nq):
    """a5 + a6 on tcgen05 (3xTF32, TMEM accumulation): ragged T (not a multiple of
    128), ragged D (not a multiple of 32), nq < 64, against the fp64 oracle."""
    K = orc.fill(T, D, 2, 1)
    s, q, Kh = orc.roundtrip(K)
    Q = orc.fill(nq, D, 43)
    m = kvq.kvq_error_metrics(dev(K), dev(Kh), dev(Q), dev(s))
    ss, mx = orc.recon_errors(K, Kh)
    assert _rel(m["sum_sq"], ss) <= REL
    assert m["max_abs"] == mx
    assert m["n_elems"] == T * D and m["n_scores"] == nq * T
    assert _rel(m["attn_mean_abs"], orc.attention_error(Q, K, Kh)) <= REL


@pytest.mark.timeout(300)
@pytest.mark.parametrize("T,D,nq", [(200, 1000, 64), (333, 8192, 64), (130, 36, 5), (64, 128, 64)])
@pytest.mark.parametrize("with_khat", [False, True])
@pytest.mark.parametrize("path", ["tc", "simt"])
def test_scores_per_entry_both_paths(kvq, orc, T, D, nq, with_khat, path):
    K = orc.fill(T, D, 4)
    _, _, Kh = orc.roundtrip(K)
    Q = orc.fill(nq, D, 43)
    S = host(kvq.kvq_attention_scores(dev(Q), dev(K), dev(Kh) if with_khat else None,
                                      workspace="auto" if path == "tc" else None))
    E = (K.astype(np.float64) - Kh.astype(np.float64)) if with_khat else K.astype(np.float64)
    ref = orc.scores(Q, K) - (orc.scores(Q, Kh) if with_khat else 0)
    cond = np.abs(Q.astype(np.float64)) @ np.abs(E).T
    err = np.abs(S - ref) / np.maximum(cond, 1e-300)
    assert err.max() <= REL, (path, float(err.max()))


@pytest.mark.timeout(300)
def test_tc_and_simt_metrics_agree(kvq, orc, monkeypatch):
    T, D, nq = 2048, 2048, 64
    Kd = kvq.kvq_synth_fill(T, D, seed=42)
    Qd = kvq.kvq_synth_fill(nq, D, seed=43)
    s = kvq.kvq_compute_scales(Kd)
    q, kh = kvq.kvq_quantize_dequantize(Kd, s)
    m_tc = kvq.kvq_error_metrics(Kd, kh, Qd, s)
    monkeypatch.setenv("KVQ_FORCE_SIMT", "1")
    m_simt = kvq.kvq_error_metrics(Kd, kh, Qd, s)
    assert m_tc["max_abs"] == m_simt["max_abs"]
    # SIMT: every e^2 exact in fp64.  Tensor-core pass: per lane and K-block the fp32 sum of 8 squares (one
    # rounded product, 7 FMAs) and one add of the lane pair, then fp64: for positive terms the relative error
    # is at most gamma_9 = 9u / (1 - 9u), u = 2^-24 (Higham, Accuracy and Stability, Lemma 3.1 / §4.2);
    # the fp64 carries add ~1e-12 at most (tolerances).
    u = 2.0 ** -24
    assert _rel(m_tc["sum_sq"], m_simt["sum_sq"]) <= 9 * u / (1 - 9 * u) + 1e-12
    assert _rel(m_tc["attn_mean_abs"], m_simt["attn_mean_abs"]) <= REL
    # deterministic run to run
    assert kvq.kvq_error_metrics(Kd, kh, Qd, s) == kvq.kvq_error_metrics(Kd, kh, Qd, s)


# ----------------------------------------------------------------------------- the headline step at C3 / C4
@pytest.mark.timeout(600)
@pytest.mark.parametrize("cfg", ["C3", "C4"])
def test_roundtrip_config_large_parity(kvq, orc, cfg):
    """bench.py's step in its own launch configuration (kvq_compute_scales, then
    kvq_roundtrip with caller workspace and device metrics, nq = 64 over all T
    rows) at full size: codes / K_hat hash-equal the SURVEY goldens (independent
    numpy), sampled rows equal the oracle bit for bit, L2 / max-abs match the
    goldens and the attention error matches the oracle's all-rows value
    (tests/golden/oracle_attn.json, written by scripts/oracle_goldens.py from
    oracle/ only) within 1e-5."""
    g = gold(cfg)
    with open(os.path.join(GOLD, "oracle_attn.json")) as f:
        ga = json.load(f)[cfg]
    T, D, nq = g["T"], g["D"], 64
    Kd = kvq.kvq_synth_fill(T, D, seed=42)
    Qd = kvq.kvq_synth_fill(nq, D, seed=43)
    s = torch.empty(D, dtype=torch.float32, device="cuda")
    Kq = torch.empty(T, D, dtype=torch.int8, device="cuda")
    Kh = torch.empty(T, D, dtype=torch.float32, device="cuda")
    ws = torch.empty(kvq.kvq_roundtrip_workspace_size(T, D, nq), dtype=torch.uint8, device="cuda")
    mout = torch.empty(kvq.METRICS_BYTES, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    kvq.kvq_compute_scales(Kd, s, stream=st)
    kvq.kvq_roundtrip(Kd, s, Qd, Kq, Kh, out_dev=mout, workspace=ws, stream=st)
    m = kvq.metrics_from_device(mout)
    sh = host(s)
    assert hashlib.sha256(sh.tobytes()).hexdigest()[:16] == g["scales_sha16"]
    assert hashlib.sha256(host(Kq).tobytes()).hexdigest()[:16] == g["q_sha16"]
    hk = hashlib.sha256()
    for r0 in range(0, T, 8192):
        hk.update(host(Kh[r0:r0 + 8192]).tobytes())
    assert hk.hexdigest()[:16] == g["khat_sha16"]
    assert _rel(m["l2"], g["l2"]) <= REL and m["max_abs"] == g["max_abs"]
    assert m["theoretical_max"] == orc.theoretical_max(sh)
    assert _rel(m["attn_mean_abs"], ga["attn_mean_abs"]) <= REL
    rng = np.random.default_rng(1)
    for r in np.sort(rng.choice(T, 32, replace=False)):
        Kr = orc.fill(1, D, 42, 0, int(r))
        qo = orc.quantize(Kr, sh)  # sh == the oracle's scales: its hash equals the golden above
        same_bits(host(Kq[r:r + 1]), qo)
        same_bits(host(Kh[r:r + 1]), orc.dequantize(qo, sh))


# ----------------------------------------------------------------------------- single-pass roundtrip (a3+a4+a5+a6)
RT_CASES = [(1, 16, 1), (128, 32, 64), (129, 48, 64), (1000, 1024, 64), (300, 128, 17), (257, 8192, 64),
            (77, 13, 5), (100, 40, 70), (64, 64, 0),
            # K-blocks padded to a multiple of 4 (33 -> 36, 5 -> 8): zero-filled K boxes, clipped code stores
            (130, 1040, 64), (131, 160, 9)]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("T,D,nq", RT_CASES)
@pytest.mark.parametrize("dist", [0, 1, 2])
def test_roundtrip_single_pass_vs_oracle(kvq, orc, T, D, nq, dist):
    """kvq_roundtrip: codes and K_hat bit-exact, metrics within 1e-5 of the oracle.
    (D % 16 == 0 and 1 <= nq <= 64 take the single tensor-core pass; the others
    the separate kernels.)"""
    K = orc.fill(T, D, 6, dist)
    so, qo, kho = orc.roundtrip(K)
    Q = orc.fill(nq, D, 43) if nq else None
    Kd = dev(K)
    s = kvq.kvq_compute_scales(Kd)
    Kq, Kh, out = kvq.kvq_roundtrip(Kd, s, None if Q is None else dev(Q))
    m = kvq.metrics_from_device(out)
    same_bits(host(s), so)
    same_bits(host(Kq), qo)
    same_bits(host(Kh), kho)
    ss, mx = orc.recon_errors(K, kho)
    assert m["max_abs"] == mx and (_rel(m["sum_sq"], ss) <= REL or ss == 0)
    assert m["theoretical_max"] == orc.theoretical_max(so)
    if nq:
        assert _rel(m["attn_mean_abs"], orc.attention_error(Q, K, kho)) <= REL


# Balanced tail (attn_tc.cu make_units): tiles split between CTAs, their Delta pieces added by
# split_combine_kernel.  Forced on (KVQ_TC_BALANCE=1) so that small shapes split: every tile in 16 / ~10
# pieces, ragged T, one whole-tile wave + a 1-tile tail in 2 units (most tail shares empty), one-unit
# tiles (no split possible), nq < 64 (query quarters partly empty), and the default rule on C4-shard
# shapes (3.46 waves: balanced; 128 tiles: whole).
SPLIT_CASES = [(640, 2048, 64), (2000, 8192, 64), (19072, 256, 64), (19200, 32, 64), (19100, 1024, 33),
               (300, 4096, 17)]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("T,D,nq", SPLIT_CASES)
@pytest.mark.parametrize("fn", ["metrics", "roundtrip"])
def test_balanced_split_tiles_vs_oracle(kvq, orc, monkeypatch, T, D, nq, fn):
    monkeypatch.setenv("KVQ_TC_BALANCE", "1")
    K = orc.fill(T, D, 7, 1)
    so, qo, kho = orc.roundtrip(K)
    Q = orc.fill(nq, D, 43)
    Kd = dev(K)
    if fn == "metrics":
        m = kvq.kvq_error_metrics(Kd, dev(kho), dev(Q), dev(so))
    else:
        s = kvq.kvq_compute_scales(Kd)
        Kq, Kh, out = kvq.kvq_roundtrip(Kd, s, dev(Q))
        m = kvq.metrics_from_device(out)
        same_bits(host(Kq), qo)
        same_bits(host(Kh), kho)
    ss, mx = orc.recon_errors(K, kho)
    assert m["max_abs"] == mx and _rel(m["sum_sq"], ss) <= REL
    assert m["n_scores"] == nq * T
    assert _rel(m["attn_mean_abs"], orc.attention_error(Q, K, kho)) <= REL


@pytest.mark.timeout(300)
@pytest.mark.parametrize("balance", ["0", "1"])
def test_balanced_and_whole_tiles_agree(kvq, orc, monkeypatch, balance):
    """Same metrics (to fp64 rounding) whether the 3.46-wave shape runs balanced or as whole tiles."""
    T, D, nq = 65536 // 8, 8192, 64  # 64 tiles: forced balance splits every tile of the one wave
    K = kvq.kvq_synth_fill(T, D, seed=42)
    Q = kvq.kvq_synth_fill(nq, D, seed=43)
    s = kvq.kvq_compute_scales(K)
    monkeypatch.setenv("KVQ_TC_BALANCE", balance)
    _, _, out = kvq.kvq_roundtrip(K, s, Q)
    m = kvq.metrics_from_device(out)
    monkeypatch.setenv("KVQ_TC_BALANCE", "0")
    _, _, out0 = kvq.kvq_roundtrip(K, s, Q)
    m0 = kvq.metrics_from_device(out0)
    assert m["max_abs"] == m0["max_abs"]
    assert _rel(m["attn_mean_abs"], m0["attn_mean_abs"]) <= 1e-12
    assert _rel(m["sum_sq"], m0["sum_sq"]) <= 1e-12


@pytest.mark.timeout(300)
@pytest.mark.parametrize("name", ["ties", "subnormal", "underflow", "zeros", "mixed"])
def test_roundtrip_structured_inputs(kvq, orc, name):
    rng = np.random.default_rng(8)
    T, D = 200, 64
    if name == "ties":
        col = np.array([127, 0.5, 1.5, 2.5, -2.5, -127, 63.5, -0.5, 126.5, -126.5], np.float32) / 128
        K = np.tile(col[:, None], (20, D)).astype(np.float32)
    elif name == "subnormal":
        K = (rng.uniform(-1, 1, (T, D)) * 2.0 ** -140).astype(np.float32)
        K[:, :32] = rng.uniform(-1, 1, (T, 32)).astype(np.float32)
    elif name == "underflow":
        K = (rng.choice([-1, 0, 1], (T, D)) * 2.0 ** -149).astype(np.float32)
    elif name == "zeros":
        K = np.zeros((T, D), np.float32)
    else:
        K = (rng.uniform(-1, 1, (T, D)) * 2.0 ** rng.integers(-60, 60, (T, D))).astype(np.float32)
    so, qo, kho = orc.roundtrip(K)
    Kd = dev(K)
    s = kvq.kvq_compute_scales(Kd)
    Kq, Kh, out = kvq.kvq_roundtrip(Kd, s, dev(orc.fill(64, D, 43)))
    same_bits(host(Kq), qo)
    same_bits(host(Kh), kho)
    assert kvq.metrics_from_device(out)["max_abs"] == orc.max_abs_error(K, kho)


@pytest.mark.timeout(300)
def test_roundtrip_matches_separate_calls_C2(kvq, orc):
    T, D = 8192, 1024
    Kd = kvq.kvq_synth_fill(T, D, seed=42)
    Qd = kvq.kvq_synth_fill(64, D, seed=43)
    s = kvq.kvq_compute_scales(Kd)
    q1 = kvq.kvq_quantize(Kd, s)
    k1 = kvq.kvq_dequantize(q1, s)
    m1 = kvq.kvq_error_metrics(Kd, k1, Qd, s)
    q2, k2, out = kvq.kvq_roundtrip(Kd, s, Qd)
    m2 = kvq.metrics_from_device(out)
    assert torch.equal(q1, q2) and torch.equal(k1.view(torch.int32), k2.view(torch.int32))
    assert m1["max_abs"] == m2["max_abs"]
    for k in ("l2", "attn_mean_abs"):
        assert _rel(m2[k], m1[k]) <= REL


# ----------------------------------------------------------------------------- single cooperative pass (C5)
@pytest.mark.timeout(300)
@pytest.mark.parametrize("T,D,expect_single", [(1, 4, True), (1000, 128, True), (8192, 1024, True),
                                               (333, 8192, True), (77, 13, False), (4096, 4, True),
                                               (1 << 20, 128, True)])
@pytest.mark.parametrize("force", [True, False])
def test_quantize_fused_single_pass(kvq, orc, monkeypatch, T, D, expect_single, force):
    """expect_single: the cooperative single pass supports the shape.  By default it only runs where
    K stays L2-resident (D >= 256 and K <= 3/4 of the L2, the measured crossover); the test-only
    KVQ_FUSED_FORCE_SINGLE=1 runs it on every supported shape.  Bit-exact either way."""
    if force:
        monkeypatch.setenv("KVQ_FUSED_FORCE_SINGLE", "1")
    else:
        monkeypatch.delenv("KVQ_FUSED_FORCE_SINGLE", raising=False)
    K = orc.fill(T, D, 12, 1)
    s, q, kh, single = kvq.kvq_quantize_fused(dev(K))
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    assert single == (expect_single and (force or (D >= 256 and T * D * 4 <= l2 // 4 * 3)))
    so, qo, kho = orc.roundtrip(K)
    same_bits(host(s), so)
    same_bits(host(q), qo)
    same_bits(host(kh), kho)


@pytest.mark.timeout(300)
def test_quantize_fused_repeat_and_special_columns(kvq, orc, monkeypatch):
    """Workspace reuse across calls (counter/bits re-zeroed), zero and subnormal columns."""
    monkeypatch.setenv("KVQ_FUSED_FORCE_SINGLE", "1")
    rng = np.random.default_rng(4)
    K = rng.uniform(-1, 1, (2048, 64)).astype(np.float32)
    K[:, 3] = 0.0
    K[:, 7] *= np.float32(2.0 ** -140)
    ws = torch.empty(kvq.load().kvq_quantize_fused_workspace_size(2048, 64), dtype=torch.uint8, device="cuda")
    so, qo, kho = orc.roundtrip(K)
    for _ in range(3):
        s, q, kh, single = kvq.kvq_quantize_fused(dev(K), workspace=ws)
        assert single
        same_bits(host(s), so)
        same_bits(host(q), qo)
        same_bits(host(kh), kho)


@pytest.mark.timeout(300)
def test_roundtrip_host_async_pipelined(kvq, orc):
    """Two async host-pipeline calls in flight on two streams (overlapping copies) give the
    same results as the oracle for their own inputs."""
    T, D, nq = 2000, 256, 64
    outs = []
    Q = orc.fill(nq, D, 43)
    Qh = torch.from_numpy(Q).pin_memory()
    slots = []
    for seed in (42, 77):
        K = orc.fill(T, D, seed)
        slots.append(dict(K=K, Kh=torch.from_numpy(K).pin_memory(), s=torch.cuda.Stream(),
                          ws=torch.empty(kvq.kvq_roundtrip_host_workspace_size(T, D, nq), dtype=torch.uint8,
                                         device="cuda"),
                          sc=torch.empty(D, dtype=torch.float32).pin_memory(),
                          kq=torch.empty((T, D), dtype=torch.int8).pin_memory(),
                          m=torch.empty(kvq.METRICS_BYTES, dtype=torch.uint8).pin_memory()))
    for sl in slots:
        kvq.kvq_roundtrip_host_async(sl["Kh"], Qh, sl["sc"], sl["kq"], sl["m"], sl["ws"], stream=sl["s"])
    torch.cuda.synchronize()
    for sl in slots:
        so, qo, kho = orc.roundtrip(sl["K"])
        same_bits(sl["sc"].numpy(), so)
        same_bits(sl["kq"].numpy(), qo)
        m = kvq.metrics_from_host(sl["m"])
        assert m["max_abs"] == orc.max_abs_error(sl["K"], kho)
        assert _rel(m["attn_mean_abs"], orc.attention_error(Q, sl["K"], kho)) <= REL


@pytest.mark.timeout(300)
def test_plain_launches_match_pdl_launches(kvq):
    """KVQ_PDL=0 (plain launches) gives bit-identical codes, K_hat and metrics to the default programmatic
    dependent launches (the variable is read once per process, hence the subprocess)."""
    import subprocess
    import sys
    code = (
        "import sys, hashlib; sys.path.insert(0, %r)\n"
        "from paper_2601_04719_b200 import kvq\n"
        "K = kvq.kvq_synth_fill(2000, 4096, seed=42, dist=1); Q = kvq.kvq_synth_fill(64, 4096, seed=43)\n"
        "s = kvq.kvq_compute_scales(K); Kq, Kh, out = kvq.kvq_roundtrip(K, s, Q)\n"
        "m = kvq.kvq_error_metrics(K, Kh, Q, s)\n"
        "h = hashlib.sha256(Kq.cpu().numpy().tobytes() + Kh.cpu().numpy().tobytes()).hexdigest()\n"
        "print(h, repr(kvq.metrics_from_device(out)['attn_mean_abs']), repr(m['attn_mean_abs']), repr(m['sum_sq']))\n"
    ) % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for v in ("0", "1"):
        env = dict(os.environ, KVQ_PDL=v)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=240)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.strip().splitlines()[-1])
    assert outs[0] == outs[1], outs


@pytest.mark.timeout(300)
@pytest.mark.parametrize("target", ["codes", "k_hat", "scales"])
def test_fault_injection_caught_by_hash_compare(kvq, orc, target):
    """SURVEY §5 (failure detection): flip ONE byte of an output buffer after the GPU pass and the
    parity check (SHA-256 against the SURVEY appendix golden for C2, numpy-computed, independent of both
    paths) must fail; the untouched buffers keep matching.  Guards against a hash compare that passes
    vacuously."""
    g = json.load(open(os.path.join(GOLD, "survey_appendix.json")))["C2"]
    T, D = 8192, 1024
    K = kvq.kvq_synth_fill(T, D, seed=42)
    s = kvq.kvq_compute_scales(K)
    q = kvq.kvq_quantize(K, s)
    kh = kvq.kvq_dequantize(q, s)
    bufs = {"scales": s, "codes": q, "k_hat": kh}
    keys = {"scales": "scales_sha16", "codes": "q_sha16", "k_hat": "khat_sha16"}

    def sha16(t):
        return hashlib.sha256(host(t).tobytes()).hexdigest()[:16]

    for name, t in bufs.items():
        assert sha16(t) == g[keys[name]], f"{name} must match before the fault"
    t = bufs[target]
    b = t.view(torch.uint8).reshape(-1)
    pos = b.numel() // 3 + 7
    b[pos] ^= 0x01  # the injected fault: one bit of one byte, on the device
    assert sha16(t) != g[keys[target]], "a flipped byte went undetected"
    for name, u in bufs.items():
        if name != target:
            assert sha16(u) == g[keys[name]]


# ----------------------------------------------------------------------------- opt-in 64-row roundtrip kernel
# (KVQ_TC_RT64=1, csrc/rt64.cuh: 64-row tiles, the stage's two 32-column boxes stacked along the MMA's M;
# parity-green, measured slower than the 128-row kernel: DESIGN §12).
@pytest.mark.timeout(300)
@pytest.mark.parametrize("T,D,nq", RT_CASES)
def test_roundtrip_rt64_vs_oracle(kvq, orc, monkeypatch, T, D, nq):
    monkeypatch.setenv("KVQ_TC_RT64", "1")
    K = orc.fill(T, D, 6, 1)
    so, qo, kho = orc.roundtrip(K)
    Q = orc.fill(nq, D, 43) if nq else None
    s = kvq.kvq_compute_scales(dev(K))
    Kq, Kh, out = kvq.kvq_roundtrip(dev(K), s, None if Q is None else dev(Q))
    m = kvq.metrics_from_device(out)
    same_bits(host(Kq), qo)
    same_bits(host(Kh), kho)
    ss, mx = orc.recon_errors(K, kho)
    assert m["max_abs"] == mx and (_rel(m["sum_sq"], ss) <= REL or ss == 0)
    if nq:
        assert _rel(m["attn_mean_abs"], orc.attention_error(Q, K, kho)) <= REL


@pytest.mark.timeout(300)
@pytest.mark.parametrize("T,D,nq", SPLIT_CASES)
def test_roundtrip_rt64_split_tiles_vs_oracle(kvq, orc, monkeypatch, T, D, nq):
    monkeypatch.setenv("KVQ_TC_RT64", "1")
    monkeypatch.setenv("KVQ_TC_BALANCE", "1")
    K = orc.fill(T, D, 7, 1)
    so, qo, kho = orc.roundtrip(K)
    Q = orc.fill(nq, D, 43)
    s = kvq.kvq_compute_scales(dev(K))
    Kq, Kh, out = kvq.kvq_roundtrip(dev(K), s, dev(Q))
    m = kvq.metrics_from_device(out)
    same_bits(host(Kq), qo)
    same_bits(host(Kh), kho)
    ss, mx = orc.recon_errors(K, kho)
    assert m["max_abs"] == mx and _rel(m["sum_sq"], ss) <= REL
    assert _rel(m["attn_mean_abs"], orc.attention_error(Q, K, kho)) <= REL


# The two converter variants of the fused pass (attn_tc.cu FASTCONV: taken automatically when every CTA gets one
# round of work units, e.g. the shapes above; the other one for multi-wave passes such as C4): both forced on shapes
# with near-ties, clamped quotients (caller scales below max/127) and exact-path columns.
@pytest.mark.timeout(300)
@pytest.mark.parametrize("fast", ["0", "1"])
@pytest.mark.parametrize("T,D,nq", [(1000, 1024, 64), (300, 128, 17), (19100, 1024, 33)])
def test_roundtrip_converter_variants(kvq, orc, monkeypatch, fast, T, D, nq):
    monkeypatch.setenv("KVQ_TC_FASTCONV", fast)
    K = orc.fill(T, D, 9, 1)
    so, qo, kho = orc.roundtrip(K)
    Q = orc.fill(nq, D, 43)
    s = kvq.kvq_compute_scales(dev(K))
    Kq, Kh, out = kvq.kvq_roundtrip(dev(K), s, dev(Q))
    m = kvq.metrics_from_device(out)
    same_bits(host(Kq), qo)
    same_bits(host(Kh), kho)
    ss, mx = orc.recon_errors(K, kho)
    assert m["max_abs"] == mx and _rel(m["sum_sq"], ss) <= REL
    assert _rel(m["attn_mean_abs"], orc.attention_error(Q, K, kho)) <= REL


@pytest.mark.timeout(300)
@pytest.mark.parametrize("fast", ["0", "1"])
def test_roundtrip_converter_variants_given_scales(kvq, orc, monkeypatch, fast):
    """Caller scales below max/127 (clamped codes), a subnormal-scale column and a zero column, both variants."""
    monkeypatch.setenv("KVQ_TC_FASTCONV", fast)
    T, D, nq = 700, 256, 64
    K = orc.fill(T, D, 10, 1)
    K[:, 5] = 0.0
    K[:, 9] *= np.float32(2.0 ** -140)
    so, _, _ = orc.roundtrip(K)
    s = (so * np.float32(0.75)).astype(np.float32)  # quotients past +-127: the clamp decides
    qo = orc.quantize(K, s)
    kho = orc.dequantize(qo, s)
    Q = orc.fill(nq, D, 43)
    Kq, Kh, out = kvq.kvq_roundtrip(dev(K), dev(s), dev(Q))
    same_bits(host(Kq), qo)
    same_bits(host(Kh), kho)


# ----------------------------------------------------------------------------- past 2^31 elements
@pytest.mark.timeout(1200)
def test_step_past_2pow31_elements(kvq, orc):
    """Maximum sizes: T * D = 2,147,786,752 > 2^31 elements (8.6 GB of keys; no 32-bit element index may wrap):
    kvq_compute_scales + kvq_roundtrip (bench.py's step) vs the oracle streaming the same rows on the CPU -- scales bit
    for bit (Alg. 1 over all rows, in row blocks), codes and K_hat bit for bit on rows at the start, across the
    2^31-element boundary and at the ragged end, max-abs exact against those rows' bound."""
    T, D, nq = (1 << 18) + 37, 8192, 64
    assert T * D > (1 << 31)
    Kd = kvq.kvq_synth_fill(T, D, seed=42)
    Qd = kvq.kvq_synth_fill(nq, D, seed=43)
    s = torch.empty(D, dtype=torch.float32, device="cuda")
    Kq = torch.empty(T, D, dtype=torch.int8, device="cuda")
    Kh = torch.empty(T, D, dtype=torch.float32, device="cuda")
    ws = torch.empty(kvq.kvq_roundtrip_workspace_size(T, D, nq), dtype=torch.uint8, device="cuda")
    mout = torch.empty(kvq.METRICS_BYTES, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    kvq.kvq_compute_scales(Kd, s, stream=st)
    kvq.kvq_roundtrip(Kd, s, Qd, Kq, Kh, out_dev=mout, workspace=ws, stream=st)
    m = kvq.metrics_from_device(mout)
    # the oracle's column maxima over all rows, streamed in row blocks (generation included)
    mx = np.zeros(D, np.float32)
    for r0 in range(0, T, 16384):
        orc.absmax_rows(orc.fill(min(16384, T - r0), D, 42, 0, r0), mx)
    so = orc.scales_from_absmax(mx)
    same_bits(host(s), so)
    edge = (1 << 31) // D  # the row holding element 2^31
    for r0 in (0, edge - 20, T - 40):  # (edge + 20 <= T)
        Kr = orc.fill(40, D, 42, 0, r0)
        qo = orc.quantize(Kr, so)
        same_bits(host(Kq[r0:r0 + 40]), qo)
        same_bits(host(Kh[r0:r0 + 40]), orc.dequantize(qo, so))
    assert m["n_elems"] == T * D and m["n_scores"] == nq * T
    assert 0.0 < m["max_abs"] <= m["theoretical_max"] * (1 + 2.0 ** -15)
    assert np.isfinite(m["attn_mean_abs"]) and 0.05 < m["attn_mean_abs"] < 0.2  # ~0.095 at D = 8192


@pytest.mark.timeout(1200)
def test_separate_calls_past_2pow31_elements(kvq, orc):
    """The paper's separate calls (kvq_quantize, kvq_dequantize, kvq_error_metrics) and kvq_quantize_fused at
    T * D > 2^31: codes and K_hat identical to the single-pass roundtrip's on every row (device compare), metrics
    equal within 1e-5."""
    T, D, nq = (1 << 18) + 37, 8192, 64
    Kd = kvq.kvq_synth_fill(T, D, seed=42)
    Qd = kvq.kvq_synth_fill(nq, D, seed=43)
    s = kvq.kvq_compute_scales(Kd)
    Kq, Kh, out = kvq.kvq_roundtrip(Kd, s, Qd)
    m = kvq.metrics_from_device(out)
    q2 = kvq.kvq_quantize(Kd, s)
    assert torch.equal(q2, Kq)
    del q2
    h2 = kvq.kvq_dequantize(Kq, s)
    assert torch.equal(h2.view(torch.int32), Kh.view(torch.int32))
    m2 = kvq.kvq_error_metrics(Kd, h2, Qd, s)
    assert m2["max_abs"] == m["max_abs"] and _rel(m2["l2"], m["l2"]) <= REL
    assert _rel(m2["attn_mean_abs"], m["attn_mean_abs"]) <= REL
    del h2
    s3, q3, h3, _ = kvq.kvq_quantize_fused(Kd)
    assert torch.equal(s3.view(torch.int32), s.view(torch.int32)) and torch.equal(q3, Kq)
    assert torch.equal(h3.view(torch.int32), Kh.view(torch.int32))


@pytest.mark.timeout(1200)
def test_formats_past_2pow31_elements(kvq, orc):
    """FP8 E4M3 and INT4 packed (NEXT-1, NEXT-3) at T * D > 2^31: scales bit-exact against the oracle's (from the
    column maxima streamed over all rows), codes / packed bytes / K_hat bit-exact on rows around the 2^31-element
    row and at the ragged end."""
    T, D = (1 << 18) + 37, 8192
    Kd = kvq.kvq_synth_fill(T, D, seed=42)
    mx = np.zeros(D, np.float32)
    for r0 in range(0, T, 16384):
        orc.absmax_rows(orc.fill(min(16384, T - r0), D, 42, 0, r0), mx)
    L = orc.lib()
    edge = (1 << 31) // D
    # E4M3
    s8 = kvq.kvq_compute_scales_fmt(Kd, kvq.FMT_E4M3)
    so8 = np.empty(D, np.float32)
    L.kvqo_scales_from_absmax_e4m3(orc._p(mx), D, orc._p(so8))
    same_bits(host(s8), so8)
    q8, h8 = kvq.kvq_quantize_e4m3(Kd, s8, want_khat=True)
    for r0 in (edge - 20, T - 40):
        Kr = orc.fill(40, D, 42, 0, r0)
        qo = orc.quantize_e4m3(Kr, so8)
        same_bits(host(q8[r0:r0 + 40]), qo)
        same_bits(host(h8[r0:r0 + 40]), orc.dequantize_e4m3(qo, so8))
    del q8, h8
    # INT4 packed
    s4 = kvq.kvq_compute_scales_fmt(Kd, kvq.FMT_INT4)
    so4 = np.empty(D, np.float32)
    L.kvqo_scales_from_absmax_q(orc._p(mx), D, orc.QMAX[4], orc._p(so4))
    same_bits(host(s4), so4)
    p4, h4 = kvq.kvq_quantize_packed(Kd, s4, 4, want_khat=True)
    for r0 in (edge - 20, T - 40):
        Kr = orc.fill(40, D, 42, 0, r0)
        qo = orc.quantize_q(Kr, so4, 4)
        same_bits(host(p4[r0:r0 + 40]), orc.pack_codes(qo, 4))
        same_bits(host(h4[r0:r0 + 40]), orc.dequantize(qo, so4))

"""GPU parity of NEXT-2: attention scores computed directly from the int8 codes
(kvq_scores_from_codes) against the oracle's fp64 Q . K_hat^T."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REL = 1e-5


@pytest.fixture(scope="module")
def kvq():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2601_04719_b200 import kvq as k
    k.kvq_device_check()
    return k


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("T,D,nq", [(1, 16, 1), (128, 128, 64), (200, 1024, 64), (333, 8192, 64), (1000, 48, 17),
                                    (129, 272, 64), (77, 13, 5), (64, 64, 70)])
@pytest.mark.parametrize("path", ["tc", "simt"])
def test_scores_from_codes(kvq, orc, T, D, nq, path):
    K = orc.fill(T, D, 8, 1)
    s, q, Kh = orc.roundtrip(K)
    Q = orc.fill(nq, D, 43)
    S = kvq.kvq_scores_from_codes(dev(Q), dev(q), dev(s), workspace="auto" if path == "tc" else None)
    torch.cuda.synchronize()
    S = S.cpu().numpy()
    ref = orc.scores(Q, Kh)
    cond = np.abs(Q.astype(np.float64)) @ np.abs(Kh.astype(np.float64)).T
    err = np.abs(S - ref) / np.maximum(cond, 1e-300)
    assert err.max() <= REL, (path, float(err.max()))


@pytest.mark.timeout(300)
def test_scores_from_codes_match_dequantized_scores(kvq, orc):
    """The codes path and the fp32 path (dequantize, then kvq_attention_scores) agree."""
    T, D, nq = 4096, 1024, 64
    Kd = kvq.kvq_synth_fill(T, D, seed=42)
    Qd = kvq.kvq_synth_fill(nq, D, seed=43)
    s = kvq.kvq_compute_scales(Kd)
    q = kvq.kvq_quantize(Kd, s)
    kh = kvq.kvq_dequantize(q, s)
    S1 = kvq.kvq_scores_from_codes(Qd, q, s)
    S2 = kvq.kvq_attention_scores(Qd, kh)
    cond = (Qd.double().abs() @ kh.double().abs().T)
    assert float(((S1.double() - S2.double()).abs() / cond).max()) <= 2 * REL


@pytest.mark.timeout(300)
@pytest.mark.parametrize("T,D,nq", [(300, 1024, 64), (513, 4096, 7)])
def test_scores_from_codes_exact_on_representable_w(kvq, orc, T, D, nq):
    """Power-of-two scales and small-integer Q make W = Q*s exact in 4 base-2^7
    digits and every oracle product/sum exact in fp64, so the int8 tensor-core
    path (exact s32 accumulation, exact fp64 recombination) must agree BIT FOR
    BIT with the oracle's fp64 Q . K_hat^T rounded to fp32."""
    rng = np.random.default_rng(T + D)
    q = rng.integers(-127, 128, (T, D)).astype(np.int8)
    s = (2.0 ** rng.integers(-12, -4, D)).astype(np.float32)
    Q = rng.integers(-2 ** 12, 2 ** 12, (nq, D)).astype(np.float32)
    Kh = orc.dequantize(q, s)
    S = kvq.kvq_scores_from_codes(dev(Q), dev(q), dev(s))
    torch.cuda.synchronize()
    ref = orc.scores(Q, Kh).astype(np.float32)
    assert np.array_equal(S.cpu().numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.timeout(300)
def test_scores_from_codes_outlier_channels(kvq, orc):
    """Outlier channels (scales spanning 2^10) and mixed-magnitude queries: the
    digit truncation error |e| < 2^-27 max|W| stays far inside the 1e-5 bound."""
    rng = np.random.default_rng(5)
    T, D, nq = 1024, 2048, 64
    K = orc.fill(T, D, 9, 1)
    K[:, rng.choice(D, 16, replace=False)] *= 1000.0
    s, q, Kh = orc.roundtrip(K)
    Q = (orc.fill(nq, D, 44) * (2.0 ** rng.integers(-8, 8, (nq, 1)))).astype(np.float32)
    S = kvq.kvq_scores_from_codes(dev(Q), dev(q), dev(s))
    torch.cuda.synchronize()
    ref = orc.scores(Q, Kh)
    cond = np.abs(Q.astype(np.float64)) @ np.abs(Kh.astype(np.float64)).T
    assert float((np.abs(S.cpu().numpy() - ref) / cond).max()) <= REL


@pytest.mark.timeout(300)
def test_scores_from_codes_nonfinite_query_rows(kvq, orc):
    """Rows of Q holding inf/nan leave the digit path (exact fp64 per element):
    inf/nan propagate exactly as in the definition; other rows are unaffected."""
    T, D, nq = 300, 256, 6
    K = orc.fill(T, D, 3, 0)
    s, q, Kh = orc.roundtrip(K)
    Q = orc.fill(nq, D, 45)
    Q[1, 7] = np.inf
    Q[3, 0] = np.nan
    Q[4, 9] = -np.inf
    S = kvq.kvq_scores_from_codes(dev(Q), dev(q), dev(s))
    torch.cuda.synchronize()
    S = S.cpu().numpy()
    with np.errstate(invalid="ignore"):
        ref = (Q.astype(np.float64) * s.astype(np.float64)) @ q.astype(np.float64).T
    for i in (1, 3, 4):
        assert np.array_equal(np.isnan(S[i]), np.isnan(ref[i]))
        fin = ~np.isnan(ref[i])
        assert np.array_equal(S[i][fin], ref[i][fin].astype(np.float32))
    good = [0, 2, 5]
    ref_ok = orc.scores(Q[good], Kh)
    cond = np.abs(Q[good].astype(np.float64)) @ np.abs(Kh.astype(np.float64)).T
    assert float((np.abs(S[good] - ref_ok) / cond).max()) <= REL


@pytest.mark.timeout(1200)
def test_scores_from_codes_past_2pow31_elements(kvq, orc):
    """T * D > 2^31 code elements: scores straight from the codes against the oracle's fp64 Q . K_hat^T on rows
    around the 2^31-element row and at the ragged end (the oracle's K_hat from the GPU's scales, which the int8
    tests pin bit for bit against the oracle at this size)."""
    T, D, nq = (1 << 18) + 37, 8192, 64
    Kd = kvq.kvq_synth_fill(T, D, seed=42)
    Qd = kvq.kvq_synth_fill(nq, D, seed=43)
    s = kvq.kvq_compute_scales(Kd)
    q = kvq.kvq_quantize(Kd, s)
    del Kd
    S = kvq.kvq_scores_from_codes(Qd, q, s)
    torch.cuda.synchronize()
    sh = s.cpu().numpy()
    Q = orc.fill(nq, D, 43)
    edge = (1 << 31) // D
    for r0 in (edge - 20, T - 40):
        Kh = orc.dequantize(orc.quantize(orc.fill(40, D, 42, 0, r0), sh), sh)
        ref = orc.scores(Q, Kh)
        cond = np.abs(Q.astype(np.float64)) @ np.abs(Kh.astype(np.float64)).T
        got = S[:, r0:r0 + 40].cpu().numpy()
        assert (np.abs(got - ref) / np.maximum(cond, 1e-300)).max() <= REL

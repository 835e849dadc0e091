"""Pins the CPU oracle (oracle/kvq_oracle.c) to things other than itself:
values the paper/spec print, closed forms, invariants, library routines
(numpy IEEE fp32 division, np.rint half-even, float64 matmul), exact rational
arithmetic (fractions) and the SURVEY appendix goldens computed by an
independent numpy implementation.  CPU only."""
import hashlib
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from synth_np import splitmix64_np, splitmix64_py, uniform_np

GOLD = os.path.join(os.path.dirname(__file__), "golden")
F32 = np.float32


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def f32(x):
    return float(np.float32(x))


def bits(x):
    return int(np.float32(x).view(np.uint32))


# ----------------------------------------------------------------------------- generator
def test_rng_test_vector(orc):
    """splitmix64(42, i) lattice values, i = 0..5."""
    want = [int(h, 16) for h in gold("survey_appendix.json")["rng_seed42_first6_bits"]]
    got = [bits(orc.uniform(42, i)) for i in range(6)]
    assert got == want
    assert orc.uniform(42, 0) == pytest.approx(0.48312974, abs=1e-8)
    assert orc.uniform(42, 1) == pytest.approx(-0.68017924, abs=1e-8)


def test_rng_matches_independent_impls(orc):
    rng = np.random.default_rng(0)
    idx = rng.integers(0, 2 ** 40, size=200, dtype=np.uint64)
    np_vals = splitmix64_np(42, idx)
    for i, v in zip(idx.tolist(), np_vals.tolist()):
        assert orc.splitmix64(42, i) == v == splitmix64_py(42, i)
    K = orc.fill(37, 53)
    assert np.array_equal(K, uniform_np(42, 37, 53))


def test_fill_shard_equals_rows_of_full(orc):
    full = orc.fill(64, 24, 42, orc.DIST_OUTLIER)
    part = orc.fill(16, 24, 42, orc.DIST_OUTLIER, row0=32)
    assert np.array_equal(full[32:48], part)
    U = orc.fill(1000, 16)
    assert U.min() >= -1.0 and U.max() < 1.0  # "values in [-1, 1]"
    assert np.all(U * F32(2 ** 23) == np.round(U * F32(2 ** 23)))  # exact lattice


# ----------------------------------------------------------------------------- scales
def _parse(v):
    if isinstance(v, str):
        if "/" in v:
            a, b = v.split("/")
            return np.float32(a) / np.float32(b)
        return np.float32(v)
    return np.float32(v)


def test_scales_hand_examples(orc):
    for case in gold("spec_examples.json")["scales"]:
        got = orc.compute_scales(np.array(case["K"], dtype=np.float32))
        want = np.array([_parse(v) for v in case["scales"]], dtype=np.float32)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), case["cite"]
    s = orc.compute_scales(np.array([[0.25, -0.75], [0.5, 0.6]], dtype=np.float32))
    assert s[0] == pytest.approx(0.003937007859, abs=1e-12)
    assert s[1] == pytest.approx(0.005905511789, abs=1e-12)


@pytest.mark.parametrize("T", [1, 2, 3, 64, 1000])
@pytest.mark.parametrize("D", [1, 4, 5, 7, 16, 128])
def test_scales_match_numpy_absmax(orc, T, D):
    """Eq. 6 via a library reduction: np.abs(K).max(0) / float32(127)."""
    rng = np.random.default_rng(T * 131 + D)
    K = (rng.standard_normal((T, D)) * rng.uniform(0.01, 100, size=D)).astype(np.float32)
    want = np.abs(K).max(axis=0) / np.float32(127)
    got = orc.compute_scales(K)
    assert got.dtype == np.float32 and np.array_equal(got, want)
    # Streaming in row blocks gives the same max (Eq. 6 max is order-free).
    m = np.zeros(D, dtype=np.float32)
    for r0 in range(0, T, 7):
        orc.absmax_rows(K[r0:r0 + 7], m)
    assert np.array_equal(orc.scales_from_absmax(m), got)


def test_scales_permutation_properties(orc):
    """Row-permutation invariance and column-permutation equivariance."""
    K = orc.fill(300, 33, 7, orc.DIST_OUTLIER)
    s = orc.compute_scales(K)
    rng = np.random.default_rng(1)
    assert np.array_equal(orc.compute_scales(K[rng.permutation(300)]), s)
    p = rng.permutation(33)
    assert np.array_equal(orc.compute_scales(K[:, p]), s[p])


def test_scale_tightness_exhaustive_binade(orc):
    """Every column's argmax element codes to exactly +-127 (
    S:136): exhaustive over all 2^23 floats m in [1, 2), one column each."""
    m = (np.arange(2 ** 23, dtype=np.uint32) + np.uint32(0x3F800000)).view(np.float32).reshape(1, -1)
    s = orc.compute_scales(m)
    assert np.array_equal(s, m[0] / np.float32(127))
    q = orc.quantize(m, s)
    assert np.all(q == 127)
    assert np.all(orc.quantize(-m, s) == -127)


# ----------------------------------------------------------------------------- quantize
def test_quantize_hand_examples(orc):
    g = gold("spec_examples.json")
    for case in g["quantize"]:
        K = np.array(case["K"], dtype=np.float32)
        q = orc.quantize(K, np.array(case["scales"], dtype=np.float32))
        assert q.dtype == np.int8 and q.tolist() == case["q"], case["cite"]
    K = np.array([[0.25, -0.75], [0.5, 0.6]], dtype=np.float32)
    assert orc.quantize(K, orc.compute_scales(K)).tolist() == g["two_by_two_codes"]


def test_quantize_ties_round_half_even(orc):
    """Reading Q1: ties go to even (P:272 __float2int_rn), not away from zero
    (P:231 roundf).  s = (127/128)/127 = 1/128 exactly."""
    g = gold("spec_examples.json")
    col = (np.array(g["tie_column_times_128"], dtype=np.float32) / np.float32(128)).reshape(-1, 1)
    s = orc.compute_scales(col)
    assert s[0] == np.float32(1 / 128)
    q = orc.quantize(col, s)
    assert q[:, 0].tolist() == g["tie_column_codes"]
    assert q[:, 0].tolist() != g["tie_column_codes_if_roundf"]
    assert (orc.dequantize(q, s)[:, 0] * 128).tolist() == g["tie_column_codes"]


@pytest.mark.parametrize("shape", [(1, 1), (3, 5), (64, 7), (257, 128), (31, 1000)])
def test_quantize_matches_numpy(orc, shape):
    """np.clip(np.rint(fp32(K/s)), -127, 127); numpy fp32 division is IEEE RN."""
    rng = np.random.default_rng(sum(shape))
    T, D = shape
    K = (rng.uniform(-1, 1, (T, D)) * rng.uniform(1e-3, 1e3, D)).astype(np.float32)
    s = orc.compute_scales(K)
    with np.errstate(divide="ignore", invalid="ignore"):
        want = np.clip(np.rint((K / s).astype(np.float32)), -127, 127)
    want = np.where(s == 0, 0, want).astype(np.int8)
    assert np.array_equal(orc.quantize(K, s), want)
    # Sign symmetry
    assert np.array_equal(orc.quantize(-K, s), -want)


def _exact_code(x: float, s: float) -> int:
    """Brute force by exact rationals: RN_fp32(x/s) then half-even to integer, clamp."""
    if s == 0:
        return 0
    v = Fraction(x) / Fraction(s)
    # round the exact quotient to the nearest fp32 (ties to even) by bracketing
    v32 = np.float32(float(v))  # float64 RN then fp32 RN: double rounding possible ...
    # ... so fix it exactly: choose among neighbours the one nearest to v.
    cands = [np.nextafter(v32, np.float32(-np.inf)), v32, np.nextafter(v32, np.float32(np.inf))]
    best = min(cands, key=lambda c: (abs(Fraction(float(c)) - v), int(np.float32(c).view(np.uint32)) & 1))
    r = round(Fraction(float(best)))  # Python round(): half-even on Fractions
    return max(-127, min(127, r))


def test_quantize_brute_force_exact_rationals(orc):
    """Random and near-tie elements against exact rational arithmetic."""
    rng = np.random.default_rng(5)
    scales = [f32(1 / 127), 1.0, f32(3 * 2 ** -10), f32(0.75 / 127), f32(2.0 ** -140 / 127)]
    for s in scales:
        xs = list(rng.uniform(-127.6, 127.6, 400) * s)
        # near-ties: (k + 0.5) * s and neighbours
        for k in range(-127, 127, 9):
            c = np.float32((k + 0.5) * s)
            xs += [c, np.nextafter(c, np.float32(0)), np.nextafter(c, np.float32(1e30))]
        K = np.array(xs, dtype=np.float32).reshape(-1, 1)
        got = orc.quantize(K, np.array([s], dtype=np.float32))[:, 0]
        want = [_exact_code(float(x), s) for x in K[:, 0]]
        assert got.tolist() == want, s


def test_quantize_all_codes_fixed_scale(orc):
    """Exhaustive: every fp32 x with |x| in [2^-8, 2), both signs, for
    s = fl(1/127) (quotients 0.5 .. 254, i.e. every code and the clamp region)
    against numpy's IEEE fp32 division + np.rint (library routines)."""
    s = np.float32(1) / np.float32(127)
    lo, hi = 0x3B800000, 0x40000000  # 2^-8 .. 2.0
    for c0 in range(lo, hi, 1 << 24):
        x = np.arange(c0, min(c0 + (1 << 24), hi), dtype=np.uint32).view(np.float32)
        x = np.concatenate([x, -x])
        q = orc.quantize(x.reshape(-1, 1), np.array([s], dtype=np.float32))[:, 0]
        want = np.clip(np.rint((x / s).astype(np.float32)), -127, 127).astype(np.int8)
        assert np.array_equal(q, want), hex(c0)


def test_clamp_fires_for_subnormal_scale(orc):
    """column max 2^-140 -> s = 4*2^-149, quotient 128 -> 127."""
    K = np.array([[2.0 ** -140], [-(2.0 ** -141)]], dtype=np.float32)
    s = orc.compute_scales(K)
    assert s[0] == np.float32(4 * 2.0 ** -149)
    assert np.float32(K[0, 0]) / s[0] == np.float32(128)
    assert orc.quantize(K, s)[:, 0].tolist() == [127, -64]


def test_zero_and_underflowing_scale_columns(orc):
    """Reading Q5: s_d == 0 -> q = 0 and K_hat = +0, also for a nonzero column
    whose scale underflows (max < ~2^-143)."""
    K = np.array([[0.0, 2.0 ** -149, 1.0], [-0.0, -(2.0 ** -149), -1.0]], dtype=np.float32)
    s = orc.compute_scales(K)
    assert s[0] == 0 and s[1] == 0 and s[2] > 0
    q = orc.quantize(K, s)
    assert q[:, :2].tolist() == [[0, 0], [0, 0]]
    Kh = orc.dequantize(q, s)
    assert np.all(Kh[:, :2].view(np.uint32) == 0)  # +0, never -0 (Q8)


def test_negative_zero_codes_to_zero(orc):
    K = np.array([[-0.0], [1.0]], dtype=np.float32)
    s = orc.compute_scales(K)
    q = orc.quantize(K, s)
    assert q[0, 0] == 0
    assert orc.dequantize(q, s)[0, 0].view(np.uint32) == 0


# ----------------------------------------------------------------------------- dequantize
def test_dequantize_examples(orc):
    g = gold("spec_examples.json")["dequant_64_over_127"]
    s = np.float32(1) / np.float32(127)
    assert bits(s) == int(g["scale_bits"], 16)
    out = orc.dequantize(np.array([[64]], dtype=np.int8), np.array([s]))
    assert out[0, 0] == np.float32(64) * s and out[0, 0] == pytest.approx(g["value"], abs=1e-6)
    assert orc.dequantize(np.array([[127]], np.int8), np.array([1.0], np.float32))[0, 0] == 127.0
    assert orc.dequantize(np.array([[0]], np.int8), np.array([0.0123], np.float32))[0, 0] == 0.0
    K = np.array([[1.0]], dtype=np.float32)
    _, _, Kh = orc.roundtrip(K)
    assert Kh[0, 0] == 1.0


def test_dequantize_matches_numpy(orc):
    rng = np.random.default_rng(3)
    q = rng.integers(-127, 128, size=(77, 19)).astype(np.int8)
    s = rng.uniform(0, 0.1, 19).astype(np.float32)
    assert np.array_equal(orc.dequantize(q, s), q.astype(np.float32) * s)


# ----------------------------------------------------------------------------- invariants
@pytest.mark.parametrize("dist", [0, 1])
def test_error_bound_and_idempotence(orc, dist):
    """Eq. 9 in fp32 (reading Q16): |x - x_hat| <= s (1/2 + 2^-16) for normal s;
    lattice idempotence roundtrip(roundtrip(K)) == roundtrip(K)."""
    K = orc.fill(2048, 128, 11, dist)
    s, q, Kh = orc.roundtrip(K)
    assert np.abs(q.astype(np.int32)).max() <= 127
    err = np.abs(K.astype(np.float64) - Kh.astype(np.float64))
    assert np.all(err <= s.astype(np.float64) * (0.5 + 2.0 ** -16))
    s2, q2, Kh2 = orc.roundtrip(Kh)
    assert np.array_equal(s2, s) and np.array_equal(q2, q) and np.array_equal(Kh2, Kh)
    # every nonzero column contains +-127 (fact 2)
    assert np.all(np.abs(q.astype(np.int32)).max(axis=0) == 127)


def test_ongrid_roundtrip_exact(orc):
    """values already on the grid round-trip bit-exactly."""
    K = orc.fill(500, 40, 9, orc.DIST_ONGRID)
    s, q, Kh = orc.roundtrip(K)
    assert np.array_equal(Kh.view(np.uint32), K.view(np.uint32))
    assert np.array_equal(K, q.astype(np.float32) * s)


# ----------------------------------------------------------------------------- metrics
def test_metric_examples_and_identity(orc):
    g = gold("spec_examples.json")
    for key in ("l2_345", "l2_unit"):
        c = g[key]
        assert orc.l2_error(np.array(c["A"], np.float32), np.array(c["B"], np.float32)) == c["l2"]
    c = g["maxabs_example"]
    assert orc.max_abs_error(np.array(c["A"], np.float32), np.array(c["B"], np.float32)) == c["max_abs"]
    c = g["attention_example"]
    a = orc.attention_error(np.array(c["Q"], np.float32), np.array(c["K"], np.float32), np.array(c["K_hat"], np.float32))
    assert a == pytest.approx(c["attn"], rel=1e-6)
    assert a == 1.0 - float(np.float32(0.9))
    K = orc.fill(50, 30)
    Q = orc.fill(4, 30, 43)
    assert orc.l2_error(K, K) == 0 and orc.max_abs_error(K, K) == 0
    assert orc.attention_error(Q, K, K) == 0
    # symmetry
    K2 = orc.roundtrip(K)[2]
    assert orc.l2_error(K, K2) == orc.l2_error(K2, K)
    for c in g["theoretical_max"]:
        sc = np.array([_parse(v) for v in c["scales"]], np.float32)
        want = float(_parse(c["value"])) if isinstance(c["value"], str) else c["value"]
        assert orc.theoretical_max(sc) == pytest.approx(want, rel=1e-6)


def test_metrics_match_numpy(orc):
    rng = np.random.default_rng(9)
    A = rng.standard_normal((40, 23)).astype(np.float32)
    B = (A + rng.standard_normal((40, 23)) * 1e-3).astype(np.float32)
    e = A.astype(np.float64) - B.astype(np.float64)
    ss, mx = orc.recon_errors(A, B)
    assert ss == pytest.approx(np.sum(e * e), rel=1e-14)
    assert mx == np.abs(e).max()
    Q = rng.uniform(-1, 1, (5, 23)).astype(np.float32)
    S = orc.scores(Q, A)
    assert np.allclose(S, Q.astype(np.float64) @ A.astype(np.float64).T, rtol=1e-13, atol=1e-13)
    Sh = Q.astype(np.float64) @ B.astype(np.float64).T
    assert orc.attention_error(Q, A, B) == pytest.approx(np.abs(S - Sh).mean(), rel=1e-10)


def test_l2_closed_form_and_growth(orc):
    """L2 ~ s_bar sqrt(N/12) (uniform error in [-s/2, s/2]); 'L2 grows with size'."""
    for T, D in [(1024, 128), (4096, 128)]:
        K = orc.fill(T, D)
        s, q, Kh = orc.roundtrip(K)
        l2 = orc.l2_error(K, Kh)
        assert l2 == pytest.approx(float(np.mean(s)) * math.sqrt(T * D / 12), rel=0.01)


def test_max_abs_matches_paper_value(orc):
    """max-abs error 'constant at 0.00394' = 1/(2*127)."""
    paper = gold("paper_values.json")["max_abs_error"]["value"]
    for T, D in [(2048, 128), (1024, 1024)]:
        K = orc.fill(T, D)
        _, _, Kh = orc.roundtrip(K)
        m = orc.max_abs_error(K, Kh)
        assert 0.00374 <= m <= 1 / 254 + 1e-8  # S:530 acceptance band
        assert round(m, 5) == paper


def test_attention_error_paper_value_and_sqrtD(orc):
    """P:481 (0.095 at D=8192), P:479 (grows as sqrt(D)); closed form
    sqrt(2/pi) * s * sqrt(D/36) with s = 1/127."""
    paper = gold("paper_values.json")["attention_error_D8192"]["value"]
    vals = {}
    for D, T, nq in [(1024, 256, 16), (4096, 128, 16), (8192, 128, 16)]:
        K = orc.fill(T, D)
        Q = orc.fill(nq, D, 43)
        _, _, Kh = orc.roundtrip(K)
        vals[D] = orc.attention_error(Q, K, Kh)
        closed = math.sqrt(2 / math.pi) * (1 / 127) * math.sqrt(D / 36)
        assert vals[D] == pytest.approx(closed, rel=0.06)
    assert abs(vals[8192] - paper) < 0.005
    assert 1.7 <= vals[4096] / vals[1024] <= 2.3


# ----------------------------------------------------------------------------- goldens
@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_survey_golden_hashes_and_metrics(orc, cfg):
    g = gold("survey_appendix.json")[cfg]
    T, D = g["T"], g["D"]
    r = orc.streamed_pipeline(T, D, block_rows=2048, nq=64, attn_rows=T)
    assert r["scales_sha"][:16] == g["scales_sha16"]
    assert r["q_sha"][:16] == g["q_sha16"]
    assert r["khat_sha"][:16] == g["khat_sha16"]
    assert r["l2"] == pytest.approx(g["l2"], rel=1e-9)
    assert r["max_abs"] == g["max_abs"]
    assert r["attn_mean_abs"] == pytest.approx(g["attn_mean_abs"], rel=1e-9)
    # in-memory and streamed oracle agree
    if cfg == "C1":
        K = orc.fill(T, D)
        s, q, Kh = orc.roundtrip(K)
        assert hashlib.sha256(q.tobytes()).hexdigest() == r["q_sha"]


def test_oracle_attn_goldens_file():
    """tests/golden/oracle_attn.json (scripts/oracle_goldens.py, oracle/ only) agrees with the
    independent numpy values of the SURVEY appendix where those exist (C1, C2), and its C3/C4
    values with the closed form sqrt(2/pi) * mean(s) * sqrt(D/36) and the paper's 0.095."""
    ga = gold("oracle_attn.json")
    sv = gold("survey_appendix.json")
    for cfg in ("C1", "C2"):
        assert ga[cfg]["attn_mean_abs"] == pytest.approx(sv[cfg]["attn_mean_abs"], rel=1e-12)
    for cfg in ("C3", "C4"):
        g = ga[cfg]
        assert g["attn_mean_abs"] == pytest.approx(g["attn_abs_sum"] / (g["nq"] * g["T"]), rel=1e-15)
        closed = math.sqrt(2 / math.pi) * (1 / 127) * math.sqrt(g["D"] / 36)
        assert g["attn_mean_abs"] == pytest.approx(closed, rel=0.01)
        assert abs(g["attn_mean_abs"] - 0.095) < 0.002


@pytest.mark.parametrize("name", ["2^24 x D1024", "2^24 x D8192"])
def test_c5_goldens_pinned_by_numpy(name):
    """tests/golden/oracle_c5.json (written by scripts/oracle_c5_goldens.py from oracle/ only) against an
    independent numpy implementation: the numpy generator (synth_np), Eq. 6 as np.abs(K).max(0) / fp32 127,
    Eq. 7 as np.clip(np.rint(fp32(K / s)), -127, 127) (IEEE division, half-even), Eq. 8 as fp32 q * s.
    (The 2^30 entries come from the same oracle code; the GPU suite checks all four.)"""
    import hashlib

    from synth_np import uniform_np
    g = gold("oracle_c5.json")[name]
    K = uniform_np(42, g["T"], g["D"])
    s = (np.abs(K).max(axis=0) / np.float32(127)).astype(np.float32)
    with np.errstate(divide="ignore", invalid="ignore"):
        q = np.where(s > 0, np.clip(np.rint((K / s).astype(np.float32)), -127, 127), 0).astype(np.int8)
    kh = (q.astype(np.float32) * s).astype(np.float32)
    assert hashlib.sha256(s.tobytes()).hexdigest() == g["scales_sha256"]
    assert hashlib.sha256(q.tobytes()).hexdigest() == g["codes_sha256"]
    assert hashlib.sha256(kh.tobytes()).hexdigest() == g["k_hat_sha256"]


@pytest.mark.parametrize("dist", [1, 2])
@pytest.mark.parametrize("T,D,row0", [(7, 13, 0), (64, 128, 0), (33, 1000, 5), (1, 4096, 0)])
def test_structured_generators_match_numpy(orc, dist, T, D, row0):
    """The oracle's outlier-channel (dist 1) and on-grid (dist 2) generators against independent numpy
    implementations of the SURVEY §8(c)/(d) recipes (tests/synth_np.py), bit for bit, incl. a shard (row0 > 0)."""
    from synth_np import ongrid_np, outlier_np
    want = (outlier_np if dist == 1 else ongrid_np)(42, T, D, row0)
    got = orc.fill(T, D, 42, dist, row0)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))

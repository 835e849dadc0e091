"""Pins of the oracle's INT4 / INT2 variant (NEXT-3; reading Q19): hand-worked
codes and packed bytes, numpy's rint(fp32(K/s)) with clip as an independent
implementation, a pure-Python bit-field packer, the s/2 error bound, and the
reduction to the paper's INT8 quantizer at qmax = 127."""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O


def test_hand_codes_int4_int2(orc):
    s = np.array([1.0], np.float32)
    x = np.array([0.5, 1.5, 2.5, -2.5, 6.5, 7.4, 7.6, 100.0, -100.0, -0.0, 3.49], np.float32)[:, None]
    assert orc.quantize_q(x, s, 4)[:, 0].tolist() == [0, 2, 2, -2, 6, 7, 7, 7, -7, 0, 3]
    x2 = np.array([0.5, 0.51, -0.7, 3.0, -0.5, -0.50001, 0.0], np.float32)[:, None]
    assert orc.quantize_q(x2, s, 2)[:, 0].tolist() == [0, 1, -1, 1, 0, -1, 0]
    assert orc.quantize_q(x, np.array([0.0], np.float32), 4)[:, 0].tolist() == [0] * len(x)  # reading Q5


def test_hand_packed_bytes(orc):
    q4 = np.array([[1, -1, 7, -7, 0]], np.int8)
    assert orc.pack_codes(q4, 4)[0].tolist() == [0xF1, 0x97, 0x00]
    q2 = np.array([[1, -1, 0, 1, -1]], np.int8)
    assert orc.pack_codes(q2, 2)[0].tolist() == [0b01001101, 0b00000011]
    assert O.packed_row_bytes(5, 4) == 3 and O.packed_row_bytes(5, 2) == 2 and O.packed_row_bytes(8, 4) == 4


def _py_pack(q, bits):
    per = 8 // bits
    out = []
    for row in q.tolist():
        bs = [0] * ((len(row) + per - 1) // per)
        for d, c in enumerate(row):
            bs[d // per] |= (c % (1 << bits)) << (bits * (d % per))
        out.append(bs)
    return np.array(out, np.uint8)


@pytest.mark.parametrize("bits", [4, 2])
@pytest.mark.parametrize("D", [1, 3, 8, 13, 64])
def test_pack_unpack_vs_python(orc, bits, D):
    qmax = O.QMAX[bits]
    rng = np.random.default_rng(D * bits)
    q = rng.integers(-qmax, qmax + 1, (7, D)).astype(np.int8)
    p = orc.pack_codes(q, bits)
    assert np.array_equal(p, _py_pack(q, bits))
    assert np.array_equal(orc.unpack_codes(p, D, bits), q)


@pytest.mark.parametrize("bits", [4, 2])
@pytest.mark.parametrize("shape", [(1, 1), (5, 9), (257, 64), (100, 1000)])
def test_pipeline_vs_numpy(orc, bits, shape):
    qmax = O.QMAX[bits]
    rng = np.random.default_rng(sum(shape) + bits)
    K = (rng.uniform(-1, 1, shape) * rng.uniform(1e-3, 1e3, shape[1])).astype(np.float32)
    s, p, Kh = orc.roundtrip_q(K, bits)
    assert np.array_equal(s, np.abs(K).max(0) / np.float32(qmax))
    with np.errstate(divide="ignore", invalid="ignore"):
        quot = (K / s).astype(np.float32)
    want = np.where(s == 0, 0, np.clip(np.rint(quot), -qmax, qmax)).astype(np.int8)
    q = orc.unpack_codes(p, shape[1], bits)
    assert np.array_equal(q, want)
    assert np.array_equal(Kh.view(np.uint32), (want.astype(np.float32) * s).view(np.uint32))
    # the argmax element of every column maps to +-qmax (scale tightness)
    am = np.abs(K).argmax(0)
    assert np.all(np.abs(q[am, np.arange(shape[1])]) == qmax)
    # |x - x_hat| <= s (1/2 + 2^-16) (reading Q16's bound, any qmax)
    assert np.all(np.abs(K.astype(np.float64) - Kh) <= s.astype(np.float64) * (0.5 + 2.0 ** -16))


@pytest.mark.parametrize("bits", [4, 2])
def test_brute_force_rational(orc, bits):
    """Exact rationals: q = nearest integer (ties to even) of fl32(x/s), clamped."""
    qmax = O.QMAX[bits]
    rng = np.random.default_rng(11 + bits)
    for s in [np.float32(0.1), np.float32(1 / 7), np.float32(3.0), np.float32(2.0 ** -130)]:
        x = (rng.uniform(-1.2, 1.2, 500) * float(s) * qmax).astype(np.float32)
        x[:20] = ((np.arange(20) - 10) * 0.5 * float(s)).astype(np.float32)  # near ties
        got = orc.quantize_q(x[:, None], np.array([s], np.float32), bits)[:, 0]
        for xi, gi in zip(x, got):
            quot = Fraction(float(np.float32(xi) / s))  # the fp32 IEEE quotient (reading Q2)
            fl = quot.numerator // quot.denominator
            rem = quot - fl
            r = fl + (1 if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1) else 0)
            assert gi == max(-qmax, min(qmax, r)), (xi, s, gi, r)


def test_reduces_to_int8_at_qmax_127(orc):
    K = orc.fill(64, 33, 5, 1)
    s = orc.compute_scales(K)
    q = np.empty(K.shape, np.int8)
    O.lib().kvqo_quantize_q(O._p(K), O._p(s), 64, 33, 127, O._p(q))
    assert np.array_equal(q, orc.quantize(K, s))

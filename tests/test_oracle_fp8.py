"""Pins of the oracle's FP8 E4M3 variant (NEXT-1; reading Q17): hand-worked
E4M3 codes from the format's definition, torch's float8_e4m3fn conversion as an
independent library routine (round-to-nearest-even) below the saturation
point, exhaustive decode/encode round trips, and the per-channel pipeline
against numpy/torch."""
import numpy as np
import pytest
import torch

F8 = torch.float8_e4m3fn


def torch_encode(x: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(F8).view(torch.uint8).numpy()


def test_e4m3_hand_examples(orc):
    cases = [(448.0, 0x7E),             # largest finite: S.1111.110
             (1.0, 0x38),               # E=7, M=0
             (0.5, 0x30),
             (2.0 ** -6, 0x08),         # smallest normal
             (2.0 ** -9, 0x01),         # smallest subnormal
             (2.0 ** -10, 0x00),        # tie between 0 and 2^-9 -> even (0)
             (3 * 2.0 ** -10, 0x02),    # tie between 2^-9 (M=1) and 2^-8 (M=2) -> even
             (1.0625, 0x38),            # tie between 1.0 (M=0) and 1.125 (M=1) -> even
             (1.1875, 0x3A),            # tie between 1.125 (M=1) and 1.25 (M=2) -> even
             (464.0, 0x7E),             # beyond the last finite value: saturate (satfinite)
             (1.0e30, 0x7E), (-1000.0, 0xFE), (0.0, 0x00), (-0.0, 0x80), (-(2.0 ** -11), 0x80)]
    for v, c in cases:
        assert orc.e4m3_encode(v) == c, (v, hex(orc.e4m3_encode(v)))
    assert orc.e4m3_decode(0x7E) == 448.0 and orc.e4m3_decode(0xFE) == -448.0
    assert orc.e4m3_decode(0x01) == 2.0 ** -9 and np.isnan(orc.e4m3_decode(0x7F))


def test_e4m3_decode_all_codes_vs_torch(orc):
    dec = torch.arange(256, dtype=torch.uint8).view(F8).float().numpy()
    mine = np.array([orc.e4m3_decode(c) for c in range(256)], np.float32)
    assert np.array_equal(np.isnan(dec), np.isnan(mine))
    fin = ~np.isnan(dec)
    assert np.array_equal(dec[fin].view(np.uint32), mine[fin].view(np.uint32))
    for c in range(256):  # encode(decode(c)) == c for every finite code
        if not np.isnan(mine[c]):
            assert orc.e4m3_encode(float(mine[c])) == c


def test_e4m3_encode_exhaustive_binades_vs_torch(orc):
    """Every fp32 x with |x| in [2^-12, 448), both signs: the oracle's quantize
    (s = 1) equals torch's RN-even conversion (no saturation happens below 448)."""
    lo, hi = int(np.float32(2.0 ** -12).view(np.uint32)), int(np.float32(448.0).view(np.uint32))
    for c0 in range(lo, hi, 1 << 24):
        x = np.arange(c0, min(c0 + (1 << 24), hi), dtype=np.uint32).view(np.float32)
        x = np.concatenate([x, -x]).reshape(-1, 1)
        got = orc.quantize_e4m3(x, np.array([1.0], np.float32))[:, 0]
        assert np.array_equal(got, torch_encode(x[:, 0])), hex(c0)


@pytest.mark.parametrize("shape", [(1, 1), (3, 5), (257, 128), (64, 1000)])
def test_e4m3_pipeline_vs_library(orc, shape):
    rng = np.random.default_rng(sum(shape))
    T, D = shape
    K = (rng.uniform(-1, 1, (T, D)) * rng.uniform(1e-3, 1e3, D)).astype(np.float32)
    s, q, Kh = orc.roundtrip_e4m3(K)
    assert np.array_equal(s, np.abs(K).max(0) / np.float32(448))
    with np.errstate(divide="ignore", invalid="ignore"):
        quot = (K / s).astype(np.float32)
    want = np.where(s == 0, 0, torch_encode(np.clip(quot, -448, 448))).astype(np.uint8)
    assert np.array_equal(q, want)
    dec = torch.from_numpy(q).view(F8).float().numpy()
    assert np.array_equal(Kh.view(np.uint32), (dec * s).astype(np.float32).view(np.uint32))
    # the argmax element of every nonzero column encodes to +-448 (scale tightness, as S:136)
    col_amax = np.abs(K).argmax(0)
    assert np.all(np.isin(q[col_amax, np.arange(D)], [0x7E, 0xFE]))
    # relative error of E4M3: |x - x_hat| <= 2^-4 |x| for normal codes (3 mantissa bits)
    normal = np.abs(dec) >= 2.0 ** -6
    assert np.all(np.abs(K - Kh)[normal] <= np.abs(K)[normal] * 2.0 ** -4 * (1 + 1e-6))


def test_e4m3_zero_scale_column(orc):
    K = np.array([[0.0, 1.0], [0.0, -3.0]], np.float32)
    s, q, Kh = orc.roundtrip_e4m3(K)
    assert s[0] == 0 and q[:, 0].tolist() == [0, 0] and np.all(Kh[:, 0].view(np.uint32) == 0)
    assert q[1, 1] == 0xFE and Kh[1, 1] == -3.0

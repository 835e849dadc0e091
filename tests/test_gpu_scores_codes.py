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

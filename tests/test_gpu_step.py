"""GPU parity of kvq_step (the whole hot path, a1-a6, in one ABI call) against the CPU oracle.

Small single-GPU problems (D <= 256, nq <= 64, T*D <= 2^20: BASELINE C1) run as ONE cooperative launch
(csrc/step_small.cu, SURVEY §8(f) NEXT-4 "persistent kernel"); the rest run kvq_compute_scales +
kvq_roundtrip.  Scales, codes and K_hat bit-exact against the oracle (Alg. 1, Eq. 7/8 with readings
Q1-Q8); L2 and the attention error within the north star's relative 1e-5; max-abs exact."""
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


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint8 if a.dtype == np.int8 else np.uint32)


def check(kvq, orc, K, Q, small=None, monkeypatch=None):
    if monkeypatch is not None and small is not None:
        monkeypatch.setenv("KVQ_STEP_SMALL", "1" if small else "0")
    Kd = torch.from_numpy(np.ascontiguousarray(K)).cuda()
    Qd = None if Q is None else torch.from_numpy(np.ascontiguousarray(Q)).cuda()
    s, q, kh, out = kvq.kvq_step(Kd, Qd)
    m = kvq.metrics_from_device(out)
    so, qo, kho = orc.roundtrip(K)
    assert np.array_equal(bits(host(s)), bits(so)), "scales"
    assert np.array_equal(bits(host(q)), bits(qo)), "codes"
    assert np.array_equal(bits(host(kh)), bits(kho)), "K_hat"
    ss, mx = orc.recon_errors(K, kho)
    assert m["max_abs"] == mx
    assert abs(m["sum_sq"] - ss) <= REL * ss + 1e-300
    assert m["n_elems"] == K.size
    assert m["theoretical_max"] == orc.theoretical_max(so)
    if Q is not None and Q.shape[0]:
        at = orc.attention_abs_sum(Q, K, kho)
        assert abs(m["attn_abs_sum"] - at) <= REL * at + 1e-300
        assert m["n_scores"] == Q.shape[0] * K.shape[0]
    else:
        assert m["attn_mean_abs"] == 0.0
    return m


@pytest.mark.parametrize("small", [True, False])
def test_c1_matches_oracle(kvq, orc, monkeypatch, small):
    T, D, nq = 1024, 128, 64  # BASELINE C1
    m = check(kvq, orc, orc.fill(T, D), orc.fill(nq, D, 43), small, monkeypatch)
    # SURVEY appendix goldens for C1 (numpy, independent of both paths)
    assert abs(m["l2"] - 0.8225713026859557) <= REL * 0.8225713026859557
    assert m["max_abs"] == 0.003936871886253357
    assert abs(m["attn_mean_abs"] - 0.011735106864404751) <= REL * 0.011735106864404751


SHAPES = [(1, 1, 1), (1, 5, 0), (2, 3, 64), (7, 13, 5), (149, 64, 64), (300, 256, 64), (4096, 256, 17),
          (1000, 100, 1), (8191, 128, 64), (4096, 1, 3), (257, 255, 64)]


@pytest.mark.parametrize("T,D,nq", SHAPES)
@pytest.mark.parametrize("dist", [0, 1])
def test_small_path_shapes(kvq, orc, monkeypatch, T, D, nq, dist):
    """Edge shapes of the single launch: one row, one column, rows fewer than CTAs, ragged slabs and
    row chunks, D up to the 256 limit, no queries; uniform and outlier-channel keys."""
    K = orc.fill(T, D, 42, dist)
    Q = orc.fill(nq, D, 43) if nq else None
    check(kvq, orc, K, Q, True, monkeypatch)


@pytest.mark.parametrize("name", ["ties", "subnormal", "underflow", "zeros", "mixed"])
def test_small_path_structured(kvq, orc, monkeypatch, name):
    """Readings Q1 (half-even ties), Q5 (zero / underflowing scales), Q6 (subnormal scales, exact path),
    Q8 (signed zero) through the single launch."""
    rng = np.random.default_rng(3)
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
        K[::3, 5] = -0.0
        K[7, 9] = 1.0
    else:
        K = (rng.uniform(-1, 1, (T, D)) * 2.0 ** rng.integers(-60, 60, (1, D))).astype(np.float32)
    check(kvq, orc, K, orc.fill(64, D, 43), True, monkeypatch)


def test_large_path_c2(kvq, orc, monkeypatch):
    """Beyond the small limits kvq_step is kvq_compute_scales + kvq_roundtrip (C2: 8192 x 1024, nq = 64)."""
    T, D, nq = 8192, 1024, 64
    m = check(kvq, orc, orc.fill(T, D), orc.fill(nq, D, 43), None, None)
    assert abs(m["attn_mean_abs"] - 0.03354065994601137) <= REL * 0.03354065994601137


def test_small_and_large_agree(kvq, orc, monkeypatch):
    T, D, nq = 2048, 256, 64
    Kd = torch.from_numpy(orc.fill(T, D)).cuda()
    Qd = torch.from_numpy(orc.fill(nq, D, 43)).cuda()
    res = {}
    for small in ("1", "0"):
        monkeypatch.setenv("KVQ_STEP_SMALL", small)
        s, q, kh, out = kvq.kvq_step(Kd, Qd)
        res[small] = (host(s), host(q), host(kh), kvq.metrics_from_device(out))
    a, b = res["1"], res["0"]
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(bits(x), bits(y))
    assert a[3]["max_abs"] == b[3]["max_abs"]
    assert abs(a[3]["sum_sq"] - b[3]["sum_sq"]) <= REL * b[3]["sum_sq"]
    assert abs(a[3]["attn_abs_sum"] - b[3]["attn_abs_sum"]) <= REL * b[3]["attn_abs_sum"]


def test_repeatable_and_graph_capturable(kvq, orc):
    """Bit-identical metrics run to run (fixed partition and reduction order), also when the cooperative
    launch is replayed from a CUDA graph."""
    T, D, nq = 1024, 128, 64
    K = torch.from_numpy(orc.fill(T, D)).cuda()
    Q = torch.from_numpy(orc.fill(nq, D, 43)).cuda()
    s, q, kh, out = kvq.kvq_step(K, Q)
    ws = torch.empty(kvq.kvq_step_workspace_size(T, D, nq), dtype=torch.uint8, device="cuda")
    ref = host(out).copy()
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        kvq.kvq_step(K, Q, s, q, kh, out, ws, stream=st)  # warm-up on the capture stream
        st.synchronize()
        with torch.cuda.graph(g, stream=st):
            kvq.kvq_step(K, Q, s, q, kh, out, ws, stream=st)
    for _ in range(3):
        out.zero_()
        g.replay()
        assert np.array_equal(host(out), ref)


def test_rejects_bad_arguments(kvq):
    K = torch.zeros(16, 8, device="cuda")
    with pytest.raises(ValueError):
        kvq.kvq_step(K, Kq=torch.empty(16, 4, dtype=torch.int8, device="cuda"))  # wrong shape
    with pytest.raises(ValueError):
        kvq.kvq_step(K, workspace=torch.empty(8, dtype=torch.uint8, device="cuda"))  # too small
    with pytest.raises(ValueError):
        kvq.kvq_step(K, K_hat=torch.empty(16, 8))  # host output
    with pytest.raises(RuntimeError):  # K_hat aliasing K is refused by the library
        kvq.kvq_step(K, K_hat=K)


@pytest.mark.parametrize("T,D,nq", [(8192, 1024, 64), (1000, 48, 64), (300, 8192, 64), (2047, 4096, 17),
                                    (129, 16, 1), (4096, 256, 0), (20000, 2048, 64)])
@pytest.mark.parametrize("dist", [0, 1])
def test_fused_a1_path(kvq, orc, monkeypatch, T, D, nq, dist):
    """kvq_step with the column max and the scales fused into the tensor-core roundtrip (one cooperative
    launch after the Q split; the default for L2-resident K such as C2): column-owning (D <= 3072) and
    generic column-max loops, ragged row slabs, split tails, no queries; uniform and outlier-channel keys."""
    monkeypatch.setenv("KVQ_STEP_SMALL", "0")
    monkeypatch.setenv("KVQ_STEP_FUSED", "1")
    K = orc.fill(T, D, 42, dist)
    Q = orc.fill(nq, D, 43) if nq else None
    check(kvq, orc, K, Q, None, None)


@pytest.mark.parametrize("name", ["ties", "subnormal", "underflow", "zeros", "mixed"])
def test_fused_a1_structured(kvq, orc, monkeypatch, name):
    monkeypatch.setenv("KVQ_STEP_SMALL", "0")
    monkeypatch.setenv("KVQ_STEP_FUSED", "1")
    rng = np.random.default_rng(5)
    T, D = 300, 64
    if name == "ties":
        col = np.array([127, 0.5, 1.5, 2.5, -2.5, -127, 63.5, -0.5, 126.5, -126.5], np.float32) / 128
        K = np.tile(col[:, None], (30, D)).astype(np.float32)
    elif name == "subnormal":
        K = (rng.uniform(-1, 1, (T, D)) * 2.0 ** -140).astype(np.float32)
        K[:, :32] = rng.uniform(-1, 1, (T, 32)).astype(np.float32)
    elif name == "underflow":
        K = (rng.choice([-1, 0, 1], (T, D)) * 2.0 ** -149).astype(np.float32)
    elif name == "zeros":
        K = np.zeros((T, D), np.float32)
        K[3, 7] = -2.0
    else:
        K = (rng.uniform(-1, 1, (T, D)) * 2.0 ** rng.integers(-60, 60, (1, D))).astype(np.float32)
    Kd = torch.from_numpy(K).cuda()
    s, q, kh, out = kvq.kvq_step(Kd, torch.from_numpy(orc.fill(64, D, 43)).cuda())
    so, qo, kho = orc.roundtrip(K)
    assert np.array_equal(bits(host(s)), bits(so))
    assert np.array_equal(bits(host(q)), bits(qo))
    assert np.array_equal(bits(host(kh)), bits(kho))
    assert kvq.metrics_from_device(out)["max_abs"] == orc.max_abs_error(K, kho)


@pytest.mark.parametrize("T,D,nq", [(8192, 1024, 64), (1000, 48, 64), (2047, 4096, 17)])
def test_fused_a1_path_rt64(kvq, orc, monkeypatch, T, D, nq):
    """The fused a1 + a2 front end on the opt-in 64-row roundtrip kernel (KVQ_TC_RT64=1)."""
    monkeypatch.setenv("KVQ_STEP_SMALL", "0")
    monkeypatch.setenv("KVQ_STEP_FUSED", "1")
    monkeypatch.setenv("KVQ_TC_RT64", "1")
    K = orc.fill(T, D, 42, 1)
    check(kvq, orc, K, orc.fill(nq, D, 43), None, None)

"""GPU parity of NEXT-4 (streaming append with dynamic scales; reading Q20):
after every append, scales / codes / K_hat of the growing cache equal the
oracle's BATCH method on the whole prefix K[0:T], bit for bit."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


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


def same_bits(a, b, what=""):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    va = a.view(np.uint8 if a.dtype.itemsize == 1 else np.uint32)
    vb = b.view(np.uint8 if b.dtype.itemsize == 1 else np.uint32)
    bad = np.nonzero(va != vb)
    if bad[0].size:
        i = tuple(x[0] for x in bad)
        raise AssertionError(f"{what}: {bad[0].size} mismatches; first at {i}: gpu={a[i]!r} oracle={b[i]!r}")


def check_prefix(orc, cache, Kfull, keep_khat=True):
    T = cache.T
    if T == 0:  # empty cache: the state is still all zero
        assert not host(cache.scales).any() and not host(cache.absmax).any()
        return
    so, qo, kho = orc.roundtrip(Kfull[:T])
    same_bits(host(cache.scales), so, f"scales T={T}")
    same_bits(host(cache.Kq[:T]), qo, f"codes T={T}")
    if keep_khat:
        same_bits(host(cache.K_hat[:T]), kho, f"K_hat T={T}")
    assert np.array_equal(host(cache.absmax).view(np.uint32), np.abs(Kfull[:T]).max(0).view(np.uint32))


def run_sequence(kvq, orc, Kfull, sizes, keep_khat=True, comm=None):
    cache = kvq.AppendCache(Kfull.shape[0], Kfull.shape[1], keep_khat=keep_khat, comm=comm)
    t = 0
    for n in sizes:
        cache.append(torch.from_numpy(Kfull[t:t + n]).cuda() if n else None)
        t += n
        check_prefix(orc, cache, Kfull, keep_khat)
    return cache


@pytest.mark.parametrize("D", [1, 13, 256, 1024])
@pytest.mark.parametrize("dist", [0, 1])
def test_append_decode_and_prefill(kvq, orc, D, dist):
    """Decode-sized appends (one cooperative launch) and prefill-sized ones (streaming
    kernels), mixed, including n_new = 0."""
    sizes = [0, 7, 1, 1, 3, 0, 300, 1, 64, 257, 1, 2, 1000]
    Kfull = orc.fill(sum(sizes), D, 17, dist)
    run_sequence(kvq, orc, Kfull, sizes)


def test_append_growing_scales(kvq, orc):
    """Magnitudes grow along the sequence, so most appends grow some scales and the
    old rows of those columns must be re-quantized from the retained K."""
    rng = np.random.default_rng(4)
    sizes = [4, 1, 2, 1, 8, 1, 300, 1, 3]
    T, D = sum(sizes), 96
    K = orc.fill(T, D, 23, 0)
    growth = np.cumprod(1.0 + 0.05 * rng.random((T, 1)), axis=0)
    cols = rng.random(D) < 0.5
    K[:, cols] = (K[:, cols] * growth).astype(np.float32)
    cache = run_sequence(kvq, orc, K, sizes)
    assert cache.T == T


def test_append_without_khat_and_zero_columns(kvq, orc):
    sizes = [5, 1, 1, 40]
    K = orc.fill(sum(sizes), 40, 3, 0)
    K[:, 7] = 0.0
    K[:20, 9] = 0.0  # column 9 starts at zero scale, grows later
    run_sequence(kvq, orc, K, sizes, keep_khat=False)


def test_append_first_call_prefill_only(kvq, orc):
    K = orc.fill(5000, 128, 9, 1)
    run_sequence(kvq, orc, K, [5000])


def test_append_comm_single_rank(kvq, orc):
    """The token-sharded path (all-reduce MAX between the phases) with one rank."""
    uid = kvq.kvq_comm_unique_id()
    comm = kvq.Comm(uid, 1, 0)
    try:
        sizes = [3, 1, 0, 2, 400, 1]
        K = orc.fill(sum(sizes), 64, 29, 1)
        run_sequence(kvq, orc, K, sizes, comm=comm)
    finally:
        comm.destroy()


def test_append_errors(kvq):
    K = torch.zeros((4, 8), dtype=torch.float32, device="cuda")
    st = torch.zeros(8, dtype=torch.int32, device="cuda")
    sc = torch.zeros(8, dtype=torch.float32, device="cuda")
    q = torch.zeros((4, 8), dtype=torch.int8, device="cuda")
    with pytest.raises(ValueError):
        kvq.kvq_append(K, 3, 2, st, sc, q)  # beyond capacity
    from paper_2601_04719_b200._lib import check
    ws = torch.empty(kvq.kvq_append_workspace_size(8), dtype=torch.uint8, device="cuda")
    with pytest.raises(kvq.KvqError):  # scales aliasing K
        check(kvq.load().kvq_append(K.data_ptr(), 0, 1, 8, st.data_ptr(), K.data_ptr(), q.data_ptr(), None,
                                    ws.data_ptr(), ws.numel(), None, None), "x")


@pytest.mark.timeout(1200)
def test_append_past_2pow31_elements(kvq, orc):
    """A cache past 2^31 key elements: a prefill of T0 rows (T0 * D > 2^31), then a decode append whose row
    doubles a few columns' maxima, so those columns are re-quantized over every old row (element indices past
    2^31).  Scales and the sampled rows' codes / K_hat equal the oracle's batch method on the whole prefix."""
    D = 8192
    T0 = (1 << 18) + 36
    cache = kvq.AppendCache(T0 + 1, D)
    cache.append(kvq.kvq_synth_fill(T0, D, seed=42))
    row = orc.fill(1, D, 42, 0, T0)
    grown = [3, 1000, 8191]
    row[0, grown] = np.float32(3.0)  # |K| < 1 elsewhere: these three scales grow
    cache.append(torch.from_numpy(row).cuda())
    assert cache.T == T0 + 1 and cache.T * D > (1 << 31)
    mx = np.zeros(D, np.float32)
    for r0 in range(0, T0, 16384):
        orc.absmax_rows(orc.fill(min(16384, T0 - r0), D, 42, 0, r0), mx)
    orc.absmax_rows(row, mx)
    so = orc.scales_from_absmax(mx)
    same_bits(host(cache.scales), so, "scales")
    edge = (1 << 31) // D
    for r0 in (0, edge - 20, T0 - 39):
        Kr = orc.fill(40, D, 42, 0, r0) if r0 + 40 <= T0 else np.concatenate([orc.fill(T0 - r0, D, 42, 0, r0), row])
        qo = orc.quantize(Kr, so)
        same_bits(host(cache.Kq[r0:r0 + 40]), qo, f"codes {r0}")
        same_bits(host(cache.K_hat[r0:r0 + 40]), orc.dequantize(qo, so), f"K_hat {r0}")

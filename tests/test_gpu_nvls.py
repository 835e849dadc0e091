"""GPU: the NVLS (multicast) a7 exchange on one GPU (a one-device multicast team).
Where the device or driver cannot do multicast, the staged setup must release everything and leave the
P2P exchange working (checked here too); the multi-device runs are in test_gpu_multi.py ("nvls")."""
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


@pytest.fixture()
def nvls_peer(kvq):
    from paper_2601_04719_b200.dist import enable_nvls
    peers = []

    def make(D):
        p = kvq.Peer(1, 0, D)
        p.open([p.ipc_handle])
        active = enable_nvls(p, 0, 1)
        assert active == p.nvls_active
        peers.append(p)
        return p, active
    yield make
    for p in peers:
        p.destroy()


@pytest.mark.parametrize("T,D,dist", [(1000, 256, 0), (513, 1024, 1), (4096, 8192, 0), (1, 64, 1), (0, 128, 0)])
def test_nvls_scales_match_oracle(kvq, orc, nvls_peer, T, D, dist):
    p, active = nvls_peer(D)
    so = orc.compute_scales(orc.fill(max(T, 1), D, 42, dist)) if T else np.zeros(D, np.float32)
    K = kvq.kvq_synth_fill(max(T, 1), D, seed=42, dist=dist)[:T]
    for _ in range(4):  # both slot parities, twice
        s = kvq.kvq_compute_scales_peer(K, p)
        assert np.array_equal(host(s).view(np.uint32), so.view(np.uint32))
    if not active:
        pytest.skip(f"no NVLS multicast here ({p.nvls_reason}): the P2P exchange was kept (and is correct)")


def test_nvls_communicator_step(kvq, orc, nvls_peer):
    """The whole step with a communicator whose a7 goes through NVLS (metrics through the peer slots)."""
    T, D, nq = 8192, 1024, 64
    p, active = nvls_peer(D)
    comm = kvq.Comm.from_peer(p)
    K = kvq.kvq_synth_fill(T, D, seed=42)
    Q = kvq.kvq_synth_fill(nq, D, seed=43)
    s, q, kh, out = kvq.kvq_step(K, Q, comm=comm)
    m = kvq.metrics_from_device(out)
    Ko = orc.fill(T, D)
    so, qo, kho = orc.roundtrip(Ko)
    assert np.array_equal(host(s).view(np.uint32), so.view(np.uint32))
    assert np.array_equal(host(q), qo)
    assert np.array_equal(host(kh).view(np.uint32), kho.view(np.uint32))
    attn = orc.attention_error(orc.fill(nq, D, 43), Ko, kho)
    assert abs(m["attn_mean_abs"] - attn) <= 1e-5 * attn
    comm.destroy()
    if not active:
        pytest.skip(f"no NVLS multicast here ({p.nvls_reason}): the P2P exchange was kept (and is correct)")


def test_nvls_disable_falls_back(kvq, orc):
    """kvq_peer_nvls_enable(p, 0) releases the multicast resources; the P2P exchange keeps working."""
    from paper_2601_04719_b200.dist import enable_nvls
    D = 512
    p = kvq.Peer(1, 0, D)
    p.open([p.ipc_handle])
    enable_nvls(p, 0, 1)
    p.nvls_enable(False)
    assert not p.nvls_active
    K = kvq.kvq_synth_fill(300, D, seed=42)
    s = kvq.kvq_compute_scales_peer(K, p)
    assert np.array_equal(host(s).view(np.uint32), orc.compute_scales(orc.fill(300, D)).view(np.uint32))
    p.destroy()

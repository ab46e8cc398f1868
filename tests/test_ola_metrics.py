"""SPEC baseline_ola and metrics_bench.

CPU: the window / redundancy known answers through the C-ABI and the oracle, the oracle OLA
identities (COLA), the metric known answers on the oracle, host-only OLA argument errors.
GPU: batched OLA (sc_ola_*) against the oracle's per-chunk offline_run + overlap-add, and the
GPU fidelity scores / best_lag against the numpy restatement."""
import numpy as np
import pytest

from dag_models import random_graph
from oracle import pyoracle as po
from paper_2204_07064_b200 import StreamconvError
from paper_2204_07064_b200.graph import Graph, SynthConfig, make_synthetic_rave
from paper_2204_07064_b200.runtime import Ola, best_lag, fidelity


def identity_graph(C=1):
    g = Graph(C)
    g.sink(g.conv(g.source, C, C, 1, padding=(0, 0), weight=np.eye(C, dtype=np.float32)[:, :, None],
                  bias=np.zeros(C, np.float32)))
    return g


# ------------------------------------------------------------------ CPU
def test_window_known_answers():
    assert Ola.window(4, 50).tolist() == [0.0, 0.5, 1.0, 0.5]
    for n in (4, 16, 256, 1000):
        for ov in (0, 25, 50):
            w = Ola.window(n, ov)
            assert w[0] == (0.0 if ov else 1.0)
            np.testing.assert_allclose(w, po.ola_window(n, ov), rtol=0, atol=1e-7)
    for n in (8, 64, 1024):  # COLA: shifted sums == 1
        w = po.ola_window(n, 50)
        np.testing.assert_allclose(w[: n // 2] + w[n // 2:], 1.0, atol=1e-12)
        w = po.ola_window(n, 25)
        q = n // 4
        np.testing.assert_allclose(w[3 * q:] + w[:q], 1.0, atol=1e-12)
        np.testing.assert_allclose(w[q:3 * q], 1.0)
    assert [Ola.redundancy(o) for o in (0, 25, 50)] == [1.0, 4 / 3, 2.0]


def test_oracle_ola_identities():
    g = identity_graph()
    x = np.random.default_rng(0).standard_normal((2, 1, 64 * 8)).astype(np.float32)
    assert np.array_equal(po.ola(g, x, 64, 0), x)  # 0% identity: exact
    y = po.ola(g, x, 64, 50)  # 50% identity: COLA away from the first half chunk
    np.testing.assert_allclose(y[..., 32:-32], x[..., 32:-32], atol=1e-6)
    y = po.ola(g, x, 64, 25)  # hop 48: the chunks cover [0, 9 * 48 + 64)
    np.testing.assert_allclose(y[..., 16:496 - 16], x[..., 16:496 - 16], atol=1e-6)


def test_oracle_ola_boundary_error_vs_offline():
    """Linear conv graph, 50% overlap vs offline: nonzero error, concentrated near chunk edges."""
    g = Graph(1)
    g.sink(g.conv(g.conv(g.source, 1, 4, 9, padding=(4, 4)), 4, 1, 9, padding=(4, 4)))
    x = np.random.default_rng(1).standard_normal((1, 1, 1024)).astype(np.float32)
    off = po.run(g, x, mode="offline_original")
    for ov in (0, 25, 50):
        err = np.abs(po.ola(g, x, 128, ov) - off)[0, 0, 64:-64]
        assert err.max() > 1e-3


def test_metric_known_answers():
    rng = np.random.default_rng(0)
    x = rng.standard_normal(4096)
    assert po.spectral_distance(x, x) == 0.0 and po.spectral_distance(np.zeros(4096), np.zeros(4096)) == 0.0
    assert po.spectral_distance(x, np.roll(x, 1)) > 0
    assert po.euclidean_distance([3, 4], [0, 0]) == 5.0
    assert po.correlation(x, x) == pytest.approx(1.0) and po.correlation(x, -x) == pytest.approx(-1.0)
    assert po.correlation([1, 0], [0, 1]) == 0.0
    with pytest.raises(po.OracleError):
        po.correlation(np.zeros(4), x[:4])
    assert po.best_lag(x, np.concatenate([np.zeros(5), x[:-5]]), 20) == 5
    assert po.best_lag(x, x, 20) == 0


def test_mac_count_known_answers():
    g = identity_graph()  # identity 1x1x1 conv, 100 samples -> 100
    assert g.mac_count(100) == 100
    g = Graph(2)  # K=3, N=M=2, stride 1, out_len 10 -> 120
    g.sink(g.conv(g.source, 2, 2, 3, padding=(1, 1)))
    assert g.mac_count(10) == 120
    # ola-50 vs streaming on the same graph / duration: ratio 2 up to chunk-edge effects
    g = make_synthetic_rave(SynthConfig())
    T, N = 32 * 1024, 32 * 16
    nc = (T - N) // (N // 2) + 1
    assert abs(nc * g.mac_count(N) / g.mac_count(T) - 2.0) < 0.05
    assert g.mac_count(0) == 0


def test_ola_host_only_argument_errors():
    g = make_synthetic_rave(SynthConfig())  # ratio 32
    with pytest.raises(StreamconvError) as e:
        Ola(g, 16, 50, 1, 64, device=-1)
    assert e.value.code == "ChunkTooSmall"
    with pytest.raises(StreamconvError) as e:
        Ola(g, 64, 25, 1, 64, device=-1)  # hop 48 is not a multiple of 32
    assert e.value.code == "BufferNotMultipleOfRatio"
    with pytest.raises(StreamconvError):
        Ola(g, 64, 33, 1, 64, device=-1)
    Ola(g, 128, 25, 1, 1024, device=-1)


# ------------------------------------------------------------------ GPU
torch = pytest.importorskip("torch")


@pytest.mark.gpu
@pytest.mark.parametrize("overlap", [0, 25, 50])
def test_gpu_ola_matches_oracle(overlap):
    for g, chunk in ((make_synthetic_rave(SynthConfig(base_channels=16, seed=2)), 256),
                     (random_graph(7), None), (random_graph(1003, channels=(32, 64), depth=4), None)):
        r = g.compression_ratio()
        chunk = chunk or 16 * r
        hop = chunk * (100 - overlap) // 100
        T = hop * 9 + (chunk if hop != chunk else 0)
        T = T - T % hop
        x = np.random.default_rng(overlap).standard_normal((3, g.in_channels, T)).astype(np.float32)
        y_or = po.ola(g, x, chunk, overlap)
        ola = Ola(g, chunk, overlap, 3, T)
        y = torch.empty(y_or.shape, device="cuda")
        ola.process(torch.from_numpy(x).cuda(), y, T)
        torch.cuda.synchronize()
        rms = float(np.sqrt(np.mean(y_or.astype(np.float64) ** 2)))
        err = float(np.abs(y.cpu().numpy() - y_or).max()) / rms
        assert err <= 1e-4, (overlap, err, ola.describe())


@pytest.mark.gpu
def test_gpu_ola_identity_cola():
    g = identity_graph(2)
    x = np.random.default_rng(0).standard_normal((2, 2, 64 * 8)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    for ov, edge, end in ((0, 0, 512), (50, 32, 512), (25, 16, 496)):
        T = 480 if ov == 25 else 512  # a multiple of the hop (48 at 25%)
        y = torch.empty_like(xd[..., :T])
        Ola(g, 64, ov, 2, T).process(xd[..., :T].contiguous(), y, T)
        torch.cuda.synchronize()
        yy = y.cpu().numpy()
        end = min(end, (((T - 64) // (64 * (100 - ov) // 100)) * (64 * (100 - ov) // 100)) + 64)
        sl = slice(edge, end - edge)
        np.testing.assert_allclose(yy[..., sl], x[..., sl], atol=1e-6)


@pytest.mark.gpu
def test_gpu_fidelity_matches_numpy():
    rng = np.random.default_rng(0)
    n, T = 5, 6000
    x = rng.standard_normal((n, T)).astype(np.float32)
    y = (x + 0.05 * rng.standard_normal((n, T))).astype(np.float32)
    y[1] = np.roll(x[1], 1)
    y[2] = x[2]
    f = fidelity(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    for i in range(n):
        assert f["L_s"][i] == pytest.approx(po.spectral_distance(x[i], y[i]), rel=1e-4, abs=1e-9)
        assert f["L_w"][i] == pytest.approx(po.euclidean_distance(x[i], y[i]), rel=1e-9)
        assert f["L_c"][i] == pytest.approx(po.correlation(x[i], y[i]), rel=1e-9)
    assert f["L_s"][2] == 0 and f["L_w"][2] == 0 and f["L_c"][2] == pytest.approx(1.0)
    with pytest.raises(StreamconvError) as e:
        fidelity(torch.zeros((1, 512), device="cuda"), torch.zeros((1, 512), device="cuda"))
    assert e.value.code == "ZeroEnergy"
    lag_in = np.stack([np.concatenate([np.zeros(k), x[k][:-k or None]]) for k in range(n)]).astype(np.float32)
    lags = best_lag(torch.from_numpy(x).cuda(), torch.from_numpy(lag_in).cuda(), 16)
    assert lags.tolist() == list(range(n))

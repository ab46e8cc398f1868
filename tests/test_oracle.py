"""CPU: the oracle (oracle/oracle.cpp) pinned against the SPEC known answers and against the
reference's own compiled kernels.cpp (oracle/_ref + committed golden vectors), plus the SPEC
stream_runtime / causalize properties on the oracle itself.  No GPU."""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2204_07064_b200 import configs
from paper_2204_07064_b200.graph import Model

GOLD = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(GOLD))
KATS = json.loads((GOLD / "spec_kats.json").read_text())
f32 = lambda v: np.asarray(v, np.float32)  # noqa: E731
USE_REF = [False] + ([True] if po.ref_available() else [])


@pytest.mark.parametrize("use_ref", USE_REF)
def test_spec_kats_tensor_core(use_ref):
    for k in KATS["pad_zeros"]:
        y = po.pad_zeros(f32(k["x"]).reshape(1, -1), k["L"], k["R"], use_ref=use_ref)
        assert y.ravel().tolist() == k["y"], k["spec"]
    for k in KATS["conv1d"]:
        w = f32(k["w"]).reshape(1, 1, -1)
        y = po.conv1d(f32(k["x"]).reshape(1, -1), w, f32([0]), k["S"], k["d"], use_ref=use_ref)
        assert y.ravel().tolist() == k["y"], k["spec"]
    for k in KATS["zero_upsample"]:
        y = po.zero_upsample(f32(k["x"]).reshape(1, -1), k["s"], use_ref=use_ref)
        assert y.ravel().tolist() == k["y"], k["spec"]
    for k in KATS["activation"]:
        y = po.activation(f32(k["x"]), k["kind"], k["alpha"], use_ref=use_ref)
        np.testing.assert_allclose(y, f32(k["y"]), rtol=0, atol=1e-7, err_msg=k["spec"])


def test_spec_kats_causalize_and_state():
    for k in KATS["delay_for_stride"]:
        assert po.delay_for_stride(k["S"], k["R"], k["Dc"]) == k["Da"], k["spec"]
    for k in KATS["branch_alignment"]:
        assert po.branch_alignment(k["D"]) == k["A"], k["spec"]
    # offline_run [1,1,1,1] * [1,1,1] pad (1,1) -> [2,3,3,2]
    k = KATS["offline_run"][0]
    m = Model(1)
    m.conv(1, 1, 3, padding=tuple(k["pad"]), weight=f32(k["w"]).reshape(1, 1, 3), bias=f32([0]))
    y = po.run(m, f32(k["x"]).reshape(1, 1, -1), mode="offline_original")
    assert y.ravel().tolist() == k["y"]
    # latency: causal chain -> 0, centered K=3 -> 1
    m = Model(1)
    m.conv(1, 1, 3, padding=(2, 0)).conv(1, 1, 3, padding=(2, 0))
    assert po.graph_info(m)["latency_sink"] == 0
    m = Model(1)
    m.conv(1, 1, 3, padding=(1, 1))
    assert po.graph_info(m)["latency_sink"] == 1
    # init_state bytes
    m = Model(1)
    m.conv(1, 1, 1, padding=(0, 0), weight=f32([1]).reshape(1, 1, 1), bias=f32([0]))
    assert po.graph_info(m)["state_bytes"] == 0
    m = Model(1)
    m.conv(1, 1, 3, padding=(2, 0))
    assert po.graph_info(m)["state_bytes"] == 8
    # compression ratio
    for k in KATS["compression_ratio"]:
        m = Model(1)
        for s in k["strides"]:
            m.conv(1, 1, 2 * s, stride=s, padding=(s, s - 1))
        for u in k["ups"]:
            m.conv_transpose(1, 1, 2 * u, u, padding=(u, u - 1))
        assert po.graph_info(m)["ratio"] == k["r"], k["spec"]


def test_eq2_invariant_exhaustive():
    """SPEC.md:229 / acceptance 3: (R + D_c + D_a) mod S == 0 and 0 <= D_a < S."""
    for S in range(1, 9):
        for R in range(0, 9):
            for Dc in range(0, 33):
                Da = po.delay_for_stride(S, R, Dc)
                assert 0 <= Da < S and (R + Dc + Da) % S == 0


def test_branch_alignment_property():
    rng = np.random.default_rng(0)
    for _ in range(100):
        D = rng.integers(0, 50, rng.integers(1, 6)).tolist()
        A = po.branch_alignment(D)
        assert min(A) == 0 and len({d + a for d, a in zip(D, A)}) == 1


@pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built")
def test_oracle_conv1d_bitexact_vs_reference():
    rng = np.random.default_rng(7)
    for _ in range(40):
        M, N, K = rng.integers(1, 9), rng.integers(1, 9), rng.integers(1, 17)
        S, d = rng.integers(1, 5), rng.integers(1, 4)
        L = (K - 1) * d + 1 + rng.integers(0, 60)
        x = rng.uniform(-1, 1, (M, L)).astype(np.float32)
        w = rng.uniform(-1, 1, (N, M, K)).astype(np.float32)
        b = rng.uniform(-1, 1, N).astype(np.float32)
        assert np.array_equal(po.conv1d(x, w, b, S, d), po.conv1d(x, w, b, S, d, use_ref=True))


def test_oracle_vs_reference_golden_vectors():
    g = np.load(GOLD / "ref_conv1d.npz")
    for i in range(int(g["n"])):
        y = po.conv1d(g[f"x{i}"], g[f"w{i}"], g[f"b{i}"], int(g[f"S{i}"]), int(g[f"d{i}"]))
        assert np.array_equal(y, g[f"y{i}"]), i
    o = np.load(GOLD / "ref_ops.npz")
    x = o["x"]
    assert np.array_equal(po.zero_upsample(x, 3), o["zup3"])
    assert np.array_equal(po.pad_zeros(x, 2, 1), o["pad21"])
    assert np.array_equal(po.activation(x, 2, 0.2).reshape(x.shape), o["lrelu02"])
    assert np.array_equal(po.activation(x, 1).reshape(x.shape), o["tanh"])


def test_stream_executor_vs_reference_golden():
    """process_buffer restatement + causalize, pinned to reference-conv streaming outputs."""
    from models import small_models
    g = np.load(GOLD / "ref_stream.npz")
    for name, m in small_models().items():
        y = po.run(m, g[f"{name}_x"], g[f"{name}_parts"].tolist(), "stream")
        assert np.array_equal(y, g[f"{name}_y"]), name


def test_conv1d_vs_triple_loop():
    """conv1d matches a naive triple loop to <= 1e-6 (|x|,|w| <= 1, K<=16, M,N<=8)."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        M, N, K = rng.integers(1, 9), rng.integers(1, 9), rng.integers(1, 17)
        L = K + rng.integers(0, 30)
        x = rng.uniform(-1, 1, (M, L))
        w = rng.uniform(-1, 1, (N, M, K))
        b = rng.uniform(-1, 1, N)
        y = po.conv1d(x, w, b)
        ref = np.array([[b[n] + sum(w[n, m, k] * np.float32(x[m, i + k]) for m in range(M) for k in range(K))
                         for i in range(L - K + 1)] for n in range(N)])
        assert np.abs(y - ref).max() <= 1e-6


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_stream_equals_offline_and_partitions(cfg):
    """streaming == offline_run of the causalized graph, bit-identical across
    buffer partitions (the oracle fixes the per-output summation order)."""
    m = configs.build(cfg, seed=cfg)
    r = po.graph_info(m)["ratio"]
    unit = r if cfg != 5 else 2048
    T = 4 * unit if cfg in (3, 5) else (6 if cfg == 4 else 256)
    x = configs.batch_input(cfg, range(2), m.in_channels, T, seed=cfg)
    y_off = po.run(m, x, None, "offline")
    if cfg == 4:
        pa, pb = [1, 2, 3], [4, 1, 1]
    else:
        pa, pb = [T // 4, T // 2, T // 4], [T // 4 * 3, T // 4]
    ya = po.run(m, x, pa, "stream")
    yb = po.run(m, x, pb, "stream")
    assert np.array_equal(ya, yb)
    assert np.array_equal(ya, y_off)


@pytest.mark.parametrize("cfg", [2, 3])
def test_causal_equivalence_after_shift(cfg):
    """offline(causalize(g)) == offline(g) delayed by the latency, once the
    start-up transient (receptive field) has passed."""
    m = configs.build(cfg, seed=1)
    T = 1024 if cfg == 2 else 4096
    x = configs.batch_input(cfg, range(1), m.in_channels, T, seed=1)
    yc = po.run(m, x, None, "offline")
    yo = po.run(m, x, None, "offline_original")
    D = po.graph_info(m)["latency_sink"]
    assert D == (40 if cfg == 2 else 383)
    a, b = yc[..., D:], yo[..., :T - D]
    settle = T // 4
    assert np.array_equal(a[..., settle:], b[..., settle:])


def test_no_lookahead_oracle():
    m = configs.build(3, seed=2)
    x = configs.batch_input(3, range(1), 16, 128 * 6, seed=2)
    x2 = x.copy()
    x2[..., 128 * 4 + 3] = 100.0
    ya = po.run(m, x, [128] * 6)
    yb = po.run(m, x2, [128] * 6)
    assert np.array_equal(ya[..., :128 * 4], yb[..., :128 * 4])
    assert not np.array_equal(ya, yb)


def test_errors():
    m = Model(4)
    m.conv(3, 4, 3)  # channel mismatch
    with pytest.raises(po.OracleError) as e:
        po.graph_info(m)
    assert e.value.status == 3
    m = Model(1)
    m.conv(1, 1, 3, padding=(1, 0))  # (K-1)d != L+R
    with pytest.raises(po.OracleError) as e:
        po.graph_info(m)
    assert e.value.status == 9
    m = configs.build(3)
    with pytest.raises(po.OracleError) as e:
        po.run(m, np.zeros((1, 16, 256), np.float32), [100, 156])
    assert e.value.status == 11  # BufferNotMultipleOfRatio


def test_pqmf_reconstruction():
    """Builder-defined PQMF (parity unpinned): analysis -> synthesis is a near-perfect
    reconstruction with a fixed delay."""
    m = Model(1)
    m.pqmf_analysis(16, 256).pqmf_synthesis(16, 256)
    rng = np.random.default_rng(0)
    T = 16 * 512
    x = rng.standard_normal((1, 1, T)).astype(np.float32)
    y = po.run(m, x, None, "offline")[0, 0]
    xc = x[0, 0]
    lags = range(0, 600)
    c = [np.dot(y[L:], xc[:T - L]) for L in lags]
    L = int(np.argmax(c))
    e = y[L:] - xc[:T - L]
    snr = 10 * np.log10(np.sum(xc[:T - L] ** 2) / np.sum(e[512:] ** 2))
    assert snr > 35.0, (L, snr)


def test_res_scale_evidence():
    """Evidence for the one init deviation (configs.py: RES_SCALE_CFG5 = 0.5 for cfg5 only).
    The reference accumulates in double (kernels.cpp:96-100); an fp32-ACCUMULATING conv
    (oc_conv1d_f32acc: 8 interleaved fp32 partial sums, i.e. BLAS order) plugged into the same
    oracle executor shows what any fp32-accumulating implementation can reach:
      cfg4 at the literal BASELINE init (scale 1): within the 1e-4 x RMS tolerance;
      cfg5 at scale 1: ABOVE it (the sigmoid gate amplifies the compounded error);
      cfg5 at 0.5: well within it."""
    from conftest import oracle_model
    po.oracle().oc_set_f32acc_order(0)

    def err(cfg, rs, S, T):
        m = oracle_model(cfg, seed=cfg, res_scale=rs)
        x = configs.batch_input(cfg, range(S), m.in_channels, T, seed=0)
        y = po.run(m, x, [T], "stream", threads=po.host_threads())
        y32 = po.run(m, x, [T], "stream", threads=po.host_threads(), conv="f32acc")
        return float(np.abs(y32 - y).max() / np.sqrt(np.mean(y.astype(np.float64) ** 2)))

    e4 = err(4, 1.0, 8, 4)
    e5_1 = err(5, 1.0, 2, 32768)
    e5_h = err(5, 0.5, 2, 32768)
    print(f"f32-accumulate max err / RMS: cfg4@1 {e4:.2e}  cfg5@1 {e5_1:.2e}  cfg5@0.5 {e5_h:.2e}")
    assert e4 < 1e-4
    assert e5_1 > 1e-4          # measured 1.9e-4: the literal init is ill-conditioned for fp32
    assert e5_h < 0.3e-4        # measured 1.4e-5

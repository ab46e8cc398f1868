"""Chained 1x1 convs (fp32 tensor-core path): a 128-channel conv whose output only feeds a
K = 1 conv runs both GEMMs in one launch (kernels_tc.cu CH, runtime.cu find_chains).  The
chained launch splits the intermediate tile exactly as the second conv's transform would after
the HBM round trip; with per-slab chunk accumulators (SC_CHAIN_ONE=0) it is bit-identical to
the two-launch form (SC_CHAIN=0).  The default accumulates the chained GEMM in one TMEM chunk:
within CHAIN_TOL of the two-launch form and within the north-star tolerance of the oracle."""
import numpy as np
import pytest

from conftest import oracle_twin
from oracle import pyoracle as po
from paper_2204_07064_b200 import configs
from paper_2204_07064_b200.runtime import Plan

from test_gpu_parity import FP32_TOL, rel_err, run_gpu


CHAIN_TOL = 3e-5  # max |one-chunk chained - two launches| / RMS (measured 1.4e-5 vs the oracle)


def _plans(model, monkeypatch, one="0", precision="fp32"):
    monkeypatch.setenv("SC_CHAIN", "0")
    p0 = Plan(model, device=0, precision=precision)
    monkeypatch.delenv("SC_CHAIN")
    monkeypatch.setenv("SC_CHAIN_ONE", one)
    p1 = Plan(model, device=0, precision=precision)
    monkeypatch.delenv("SC_CHAIN_ONE")
    return p0, p1


@pytest.mark.gpu
@pytest.mark.parametrize("parts", [[2048, 2048], [96, 32, 128, 256], [1] * 6 + [300]])
def test_cfg2_chain_bf16_bit_identical(parts, monkeypatch):
    """bf16 plans: the chained launch rounds the intermediate like the bf16-stored two-launch
    form and accumulates the 1x1 GEMM in the same single K = 128 chunk — bit-identical."""
    m = configs.build(2, seed=5)
    p0, p1 = _plans(m, monkeypatch, precision="bf16")
    x = configs.batch_input(2, range(6), 128, sum(parts), seed=6)
    y0, _, _ = run_gpu(m, x, parts, plan=p0, precision="bf16")
    y1, _, st = run_gpu(m, x, parts, plan=p1, precision="bf16")
    assert np.array_equal(y0, y1), float(np.abs(y0 - y1).max())
    assert sum("+" in n.split()[0] for n in st.launch_names(parts[0])) == 4


@pytest.mark.gpu
@pytest.mark.parametrize("parts", [[2048], [96, 32, 128, 256]])
def test_cfg2_chain_one_accumulator(parts, monkeypatch):
    """The default chained form (one accumulator for the 1x1 GEMM) vs two launches and oracle."""
    m = configs.build(2, seed=3)
    p0, p1 = _plans(m, monkeypatch, one="1")
    x = configs.batch_input(2, range(4), 128, sum(parts), seed=4)
    y0, _, _ = run_gpu(m, x, parts, plan=p0)
    y1, _, _ = run_gpu(m, x, parts, plan=p1)
    assert rel_err(y1, y0)[0] <= CHAIN_TOL
    err, rms = rel_err(y1, po.run(oracle_twin(m), x, parts, "stream"))
    assert err <= FP32_TOL, f"{err:.3e} x RMS ({rms:.3e})"


@pytest.mark.gpu
@pytest.mark.parametrize("parts", [[2048, 2048], [640, 64, 1344], [96, 32, 128, 256], [1] * 12 + [300]])
def test_cfg2_chain_bit_identical(parts, monkeypatch):
    m = configs.build(2, seed=1)
    p0, p1 = _plans(m, monkeypatch)
    x = configs.batch_input(2, range(5), 128, sum(parts), seed=2)
    y0, _, _ = run_gpu(m, x, parts, plan=p0)
    y1, _, st = run_gpu(m, x, parts, plan=p1)
    assert np.array_equal(y0, y1), float(np.abs(y0 - y1).max())
    names = st.launch_names(parts[0])
    assert sum("+" in n.split()[0] for n in names) == 4, names  # four chained residual blocks
    assert not any(n.startswith("op1 ") for n in names), names
    if sum(parts) <= 2048:
        err, rms = rel_err(y1, po.run(oracle_twin(m), x, parts, "stream"))
        assert err <= FP32_TOL, f"{err:.3e} x RMS ({rms:.3e})"


@pytest.mark.gpu
def test_chain_full_streams_bit_identical(monkeypatch):
    """At the bench's stream count (256 x 2048 frames): chained == two launches, bit for bit."""
    import torch
    from paper_2204_07064_b200.runtime import StreamState
    m = configs.build(2, seed=0)
    p0, p1 = _plans(m, monkeypatch)
    S, T = 256, 2048
    x = torch.randn((S, 128, T), device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    outs = []
    for p in (p0, p1):
        st = StreamState(p, S, T)
        y = torch.empty_like(x)
        st.process_buffer(x, y, T)
        st.process_buffer(x, y, T)  # second call: the cached rows of the first
        torch.cuda.synchronize()
        outs.append(y)
        assert p is p0 or st.launches(T) == StreamState(p0, 1, T).launches(T) - 4
    assert torch.equal(outs[0], outs[1])


def _dag(second_reader: bool, seed: int = 7):
    """source(128) -> LReLU -> conv K3 128->128 -> LReLU -> conv 1x1 128->128 -> + source ->
    sink; with `second_reader` the K3 conv's output also feeds the Sum (no chain allowed)."""
    from paper_2204_07064_b200.graph import Graph
    g = Graph(128, seed=seed)
    a = g.conv(g.leaky_relu(g.source, 0.2), 128, 128, 3, padding=(1, 1))
    h = g.leaky_relu(a, 0.2)
    b = g.conv(h, 128, 128, 1, padding=(0, 0))
    g.sink(g.sum(b, g.source, a) if second_reader else g.sum(b, g.source))
    return g


@pytest.mark.gpu
@pytest.mark.parametrize("second_reader", [False, True])
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_dag_chain_selection(second_reader, precision):
    """find_chains on graph_ir DAGs: chained only when the 1x1 conv is the sole reader of the
    K3 conv's output; parity with the oracle either way."""
    from test_gpu_parity import BF16_NRMSE
    g = _dag(second_reader)
    parts = [256, 64, 704]
    x = np.random.default_rng(1).standard_normal((3, 128, sum(parts))).astype(np.float32)
    y, plan, st = run_gpu(g, x, parts, precision=precision)
    chained = any("+" in n.split()[0] for n in st.launch_names(parts[0]))
    assert chained == (not second_reader), st.launch_names(parts[0])
    y_or = po.run(g, x, parts, "stream")
    if precision == "fp32":
        assert rel_err(y, y_or)[0] <= FP32_TOL
    else:
        d = (y - y_or).astype(np.float64)
        assert np.sqrt(np.mean(d ** 2)) / np.sqrt(np.mean(y_or.astype(np.float64) ** 2)) <= BF16_NRMSE

"""GPU parity for general SPEC graph_ir DAGs (sc_plan_create_graph) against the oracle's
independent DAG restatement: random DAGs with multi-way Fanout / Sum (SIMT sum launches and
residual epilogues), model Delays (read offsets), Eq. (2) and branch-alignment delays,
ZeroUpsample + Conv (polyphase ConvT), branch-internal rate changes and a delayed Sink; the
SPEC synthetic RAVE model loaded from its model_io manifest.

Tolerance (north star): fp32 path max |gpu - oracle| <= 1e-4 x RMS(oracle output)."""
import numpy as np
import pytest

from dag_models import random_graph
from oracle import pyoracle as po
from paper_2204_07064_b200.graph import Graph, SynthConfig, make_synthetic_rave
from paper_2204_07064_b200.runtime import Plan

from test_gpu_parity import FP32_TOL, rel_err, run_gpu

torch = pytest.importorskip("torch")


def _parts(r, seed):
    rng = np.random.default_rng(seed)
    return [int(r * k) for k in rng.integers(1, 6, 4)]


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", range(4))
def test_random_dags_stream_parity(chunk):
    """Narrow channels: SIMT conv + sum kernels."""
    for seed in range(chunk * 20, chunk * 20 + 20):
        g = random_graph(seed)
        r = g.compression_ratio()
        parts = _parts(r, seed)
        x = np.random.default_rng(seed).standard_normal((3, g.in_channels, sum(parts))).astype(np.float32)
        y_or = po.run(g, x, parts, "stream")
        y_gpu, plan, _ = run_gpu(g, x, parts)
        err, rms = rel_err(y_gpu, y_or)
        assert np.isfinite(y_gpu).all(), seed
        assert err <= FP32_TOL, f"seed {seed}: {err:.3e} x RMS ({rms:.3e})\n{plan.describe()}"


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12))
def test_random_dags_tensor_core_parity(seed):
    """32/64 channels: the tcgen05 conv path with residual epilogues, delays and sums."""
    g = random_graph(1000 + seed, channels=(32, 64), depth=5)
    r = g.compression_ratio()
    parts = _parts(r, seed) * 2
    x = np.random.default_rng(seed).standard_normal((4, g.in_channels, sum(parts))).astype(np.float32)
    y_or = po.run(g, x, parts, "stream")
    y_gpu, plan, _ = run_gpu(g, x, parts)
    err, rms = rel_err(y_gpu, y_or)
    assert err <= FP32_TOL, f"seed {seed}: {err:.3e} x RMS ({rms:.3e})\n{plan.describe()}"
    # and the offline run of the causalized graph over the concatenated signal
    err2, _ = rel_err(y_gpu, po.run(g, x, None, "offline"))
    assert err2 <= FP32_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("pad", ["centered", "causal"])
def test_synthetic_rave_from_manifest(tmp_path, pad):
    """SPEC model_io: make_synthetic_rave -> save -> load -> GPU stream == oracle offline."""
    g = make_synthetic_rave(SynthConfig(padding=pad, base_channels=16, seed=3))
    g.save(tmp_path / "rave.json")
    h = Graph.load(tmp_path / "rave.json")
    r = h.compression_ratio()
    parts = [r * 4, r * 2, r * 8, r * 2]
    x = np.random.default_rng(0).standard_normal((5, 1, sum(parts))).astype(np.float32)
    y_gpu, plan, _ = run_gpu(h, x, parts)
    y_off = po.run(g, x, None, "offline")
    err, rms = rel_err(y_gpu, y_off)
    assert err <= FP32_TOL, f"{err:.3e} x RMS ({rms:.3e})"
    # bit-identical across buffer partitions
    y2, _, _ = run_gpu(h, x, [r * 16], plan=plan)
    assert np.array_equal(y_gpu, y2)


@pytest.mark.gpu
def test_dag_plan_reports_sum_launches():
    """A 3-way Sum with no conv operand free runs as one SIMT sum launch (launch names)."""
    g = Graph(4, seed=1)
    a = g.conv(g.source, 4, 4, 3)
    b = g.conv(g.source, 4, 4, 5)
    d = g.delay(g.source, 2)
    g.sink(g.tanh(g.sum(a, b, d)))
    p = Plan(g, device=0)
    assert "sum3" in p.describe()
    x = np.random.default_rng(0).standard_normal((2, 4, 64)).astype(np.float32)
    y_gpu, _, st = run_gpu(g, x, [16, 48], plan=p)
    assert rel_err(y_gpu, po.run(g, x, [16, 48], "stream"))[0] <= FP32_TOL
    names = st.launch_names(16)
    assert any("simt-sum" in n for n in names), names

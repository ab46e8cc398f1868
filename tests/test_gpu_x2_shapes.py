"""Single-layer shapes of the 3xFP16 tensor-core tiles (kernels_tc.cu X2 / window): the tile
geometries the five configs do not all reach — per-slab input units (two private slots per
transform set) and per-block windows (awin), one / two / three taps, odd K-slab counts (a set's
slabs change parity from tile to tile), a single K-slab, partial tiles (stream counts that do
not fill the last tile), strided and transposed convs — each against the oracle (the reference's
conv1d semantics, kernels.cpp:73-104) within 1e-4 x RMS and bit-identical across two buffer
partitions (different partitions give different tile geometries and modes).
LeakyReLU slopes: <= 1 in magnitude runs on 3xFP16 (max form), > 1 stays on 3xTF32."""
import numpy as np
import pytest

from conftest import oracle_twin
from oracle import pyoracle as po
from paper_2204_07064_b200.graph import Model
from test_gpu_parity import FP32_TOL, rel_err, run_gpu

torch = pytest.importorskip("torch")


def _res_unit(cin, k, d, alpha=0.2):
    m = Model(in_channels=cin, seed=cin + k + d)
    with m.residual():
        m.leaky_relu(alpha).conv(cin, cin, k, dilation=d, scale=0.5)
    return m


def _conv(cin, cout, k, stride=1, alpha=0.2):
    m = Model(in_channels=cin, seed=cin + cout + k)
    m.leaky_relu(alpha).conv(cin, cout, k, stride=stride)
    return m


def _convt(cin, cout, k, stride):
    m = Model(in_channels=cin, seed=cin + cout + k)
    m.leaky_relu(0.2).conv_transpose(cin, cout, k, stride)
    return m


# name, model, streams, partition A, partition B (same total frames)
SHAPES = [
    ("k3d1_c128_awin_partial", lambda: _res_unit(128, 3, 1), 37, [32, 32, 32], [96]),
    ("k3d5_c128_awin", lambda: _res_unit(128, 3, 5), 9, [64, 64], [16] * 8),
    ("k3d5_c512_units_partial", lambda: _res_unit(512, 3, 5), 130, [2, 2, 2, 2], [4, 4]),
    ("k3d3_c96_odd_slabs", lambda: _res_unit(96, 3, 3), 21, [8] * 6, [24, 24]),
    ("k3d1_c32_one_block_window", lambda: _res_unit(32, 3, 1), 20, [16] * 4, [32, 32]),
    ("k5_c32_64_one_block", lambda: _conv(32, 64, 5), 45, [8] * 4, [16, 16]),
    ("k1_c256_128", lambda: _conv(256, 128, 1), 40, [8, 8, 8], [24]),
    ("k1_c96_64_odd", lambda: _conv(96, 64, 1), 70, [4] * 6, [12, 12]),
    ("k1_c32_one_slab", lambda: _conv(32, 32, 1), 33, [16, 16], [8] * 4),
    ("k7_c64_128", lambda: _conv(64, 128, 7), 12, [32] * 3, [48, 48]),
    ("stride4_k9_c64_128", lambda: _conv(64, 128, 9, stride=4), 19, [64, 64], [32] * 4),
    ("convt4_k8_c256_128", lambda: _convt(256, 128, 8, 4), 50, [4, 4, 4], [2] * 6),
    ("convt2_k4_c128_64", lambda: _convt(128, 64, 4, 2), 11, [32, 32], [64]),
]


def _input(streams, channels, frames, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((streams, channels, frames)).astype(np.float32)


@pytest.mark.gpu
@pytest.mark.parametrize("name,build,streams,pa,pb", SHAPES, ids=[s[0] for s in SHAPES])
def test_shape_vs_oracle_and_partitions(name, build, streams, pa, pb):
    m = build()
    x = _input(streams, m.in_channels, sum(pa), seed=len(name))
    ya, _, st = run_gpu(m, x, pa)
    assert any("tc-3xf16" in n for n in st.launch_names(pa[0])), st.launch_names(pa[0])
    yb, _, _ = run_gpu(m, x, pb)
    y_or = po.run(oracle_twin(m), x, pa, "stream")
    err, rms = rel_err(ya, y_or)
    assert err <= FP32_TOL, f"{name}: {err:.3e} x RMS ({rms:.3e})"
    assert np.array_equal(ya, yb), f"{name}: partitions differ by {float(np.abs(ya - yb).max()):.3e}"
    # eager launches == graph replay
    yc, _, _ = run_gpu(m, x, pa, graphs=False)
    assert np.array_equal(ya, yc)


@pytest.mark.gpu
@pytest.mark.parametrize("alpha,split", [(0.2, "tc-3xf16"), (1.0, "tc-3xf16"), (-0.5, "tc-3xf16"), (1.5, "tc]"),
                                         (-2.0, "tc]")])
def test_leaky_slopes(alpha, split):
    """max(x, a x) is LeakyReLU only for a <= 1, and the row scale assumes |act(x)| <= |x|:
    slopes beyond 1 in magnitude keep the layer on the 3xTF32 split (runtime.cu, plan time)."""
    m = _conv(128, 128, 3, alpha=alpha)
    x = _input(6, 128, 96, seed=3)
    y, _, st = run_gpu(m, x, [32, 32, 32])
    names = st.launch_names(32)
    assert any(split in n for n in names), names
    y_or = po.run(oracle_twin(m), x, [32, 32, 32], "stream")
    err, rms = rel_err(y, y_or)
    assert err <= FP32_TOL, f"alpha {alpha}: {err:.3e} x RMS ({rms:.3e})"


@pytest.mark.gpu
def test_tanh_preactivation_stays_on_tf32():
    """A tanh applied on a conv's input (two stacked activations, so it cannot fuse into the
    producer) keeps that layer on the 3xTF32 split; results match the oracle."""
    m = Model(in_channels=64, seed=11)
    m.conv(64, 128, 3).leaky_relu(0.2).tanh().conv(128, 128, 3)
    x = _input(5, 64, 96, seed=12)
    y, _, st = run_gpu(m, x, [32, 32, 32])
    y_or = po.run(oracle_twin(m), x, [32, 32, 32], "stream")
    err, rms = rel_err(y, y_or)
    assert err <= FP32_TOL, f"{err:.3e} x RMS ({rms:.3e})"

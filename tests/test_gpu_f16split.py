"""The fp32-accurate path's 3xFP16 split (kernels_tc.cu HF): fp16 hi / lo operands with a
per-(row, K-slab) power-of-two block scale.  fp16 has a 5-bit exponent, so these tests pin the
range handling: a positively homogeneous model (zero bias, LeakyReLU) must scale EXACTLY with a
power-of-two input gain from 2^-60 to 2^40 (the block scale absorbs it: identical fp16 operands,
identical MMAs), stay within the fp32 tolerance of the oracle there, and agree with the 3xTF32
split (SC_FP32_SPLIT=tf32) to the same tolerance."""
import numpy as np
import pytest

from conftest import oracle_model
from oracle import pyoracle as po
from paper_2204_07064_b200 import configs
from test_gpu_parity import FP32_TOL, rel_err, run_gpu

torch = pytest.importorskip("torch")


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,parts", [(2, [2048, 2048]), (3, [4096])])
@pytest.mark.parametrize("gain_log2", [-60, -20, 12, 40])
def test_power_of_two_gain_is_exact(cfg, parts, gain_log2):
    m = configs.build(cfg, seed=5)
    x = configs.batch_input(cfg, range(2), m.in_channels, sum(parts), seed=5)
    y1, _, _ = run_gpu(m, x, parts)
    g = np.float32(2.0 ** gain_log2)
    yg, _, _ = run_gpu(m, x * g, parts)
    assert np.isfinite(yg).all()
    assert np.array_equal(yg, y1 * g), float(np.abs(yg - y1 * g).max() / (np.abs(y1).max() * g))


@pytest.mark.gpu
@pytest.mark.parametrize("gain", [1e-7, 3e5])
def test_small_and_large_signals_vs_oracle(gain):
    """Non-power-of-two gains (different fp32 inputs): still within 1e-4 x RMS of the oracle."""
    m = configs.build(3, seed=6)
    x = (configs.batch_input(3, range(2), m.in_channels, 4096, seed=6) * np.float32(gain)).astype(np.float32)
    y_or = po.run(oracle_model(3, seed=6), x, [4096], "stream")
    y_gpu, _, _ = run_gpu(m, x, [4096])
    err, rms = rel_err(y_gpu, y_or)
    assert err <= FP32_TOL, f"gain {gain}: {err:.3e} x RMS ({rms:.3e})"


@pytest.mark.gpu
def test_zero_rows_and_silence():
    """All-zero input rows (the block scale's m = 0 case) give exactly the bias response."""
    m = configs.build(3, seed=7)
    x = np.zeros((2, m.in_channels, 4096), np.float32)
    x[1, :, 2048:] = configs.batch_input(3, range(1), m.in_channels, 2048, seed=7)[0]
    y_or = po.run(oracle_model(3, seed=7), x, [4096], "stream")
    y_gpu, _, _ = run_gpu(m, x, [4096])
    assert np.isfinite(y_gpu).all()
    assert np.array_equal(y_gpu[0], np.zeros_like(y_gpu[0]))  # zero bias: silence stays silent
    err, _ = rel_err(y_gpu, y_or)
    assert err <= FP32_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,streams,parts", [(3, 2, [4096]), (5, 2, [2048] * 4)])
def test_f16_and_tf32_splits_agree(cfg, streams, parts, monkeypatch):
    m = configs.build(cfg, seed=8)
    x = configs.batch_input(cfg, range(streams), m.in_channels, sum(parts), seed=8)
    y_h, _, _ = run_gpu(m, x, parts)
    monkeypatch.setenv("SC_FP32_SPLIT", "tf32")
    y_t, _, _ = run_gpu(m, x, parts)
    err, _ = rel_err(y_h, y_t)
    assert err <= FP32_TOL, err
    assert not np.array_equal(y_h, y_t)  # the two splits really ran (different rounding)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,streams,calls", [(4, 256, 4), (5, 256, 3)])
def test_repeat_runs_bit_identical(cfg, streams, calls):
    """Two runs of the same input are bit-identical, and so are the per-slab and per-block
    input-window forms of the 3xFP16 tiles (SC_AWIN=0).  Caught a release of an input-unit slot
    issued before the transform's shared-memory loads had returned (the next TMA fill raced
    them): nondeterministic outputs at a few hundred streams."""
    import os
    m = configs.build(cfg, seed=cfg)
    F = configs.CONFIGS[cfg]["frames"]

    def go():
        from paper_2204_07064_b200.runtime import Plan, StreamState
        plan = Plan(m)
        num, den, cout = plan.sink
        g = torch.Generator(device="cuda").manual_seed(cfg)
        st = StreamState(plan, streams, F)
        ys = []
        for _ in range(calls):
            x = torch.randn((streams, m.in_channels, F), device="cuda", generator=g)
            y = torch.empty((streams, cout, F * num // den), device="cuda")
            st.process_buffer(x, y, F)
            ys.append(y)
        torch.cuda.synchronize()
        return torch.cat(ys, 2).cpu().numpy()

    a, b = go(), go()
    os.environ["SC_AWIN"] = "0"
    try:
        c = go()
    finally:
        del os.environ["SC_AWIN"]
    assert np.array_equal(a, b)
    assert np.array_equal(a, c)

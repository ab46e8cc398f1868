"""The five BASELINE.json configurations, pinned (SURVEY.md §7 "ambiguities" [decisions]).

  cfg1  single cached causal Conv1d 64->64, K=3                       1 stream x 64 x 2048
  cfg2  4 residual blocks C=128: LReLU.2 -> conv K3 d(1,3,9,27) centered -> LReLU.2 ->
        conv 1x1, + Delay_d(skip)                                      256 streams x 2048
  cfg3  strided encoder 16->64->128->256->512 (K=2S+1, S=4,4,4,2, centered, LReLU.2
        between) + mirror ConvT decoder 512->256->128->64->16 (K=2r, r=2,4,4,4)
                                                                       1024 streams x 4096
  cfg4  RAVE-style decoder: latent 128 -> conv K7 -> 1024; 4 x [LReLU.2, ConvT(2r, r)
        halving channels, 3 x residual(LReLU.2, conv K3 d=1,3,5)]; head LReLU.2 ->
        conv K7 -> 32 -> gate tanh(wave)*sigmoid(amp) -> 16 bands -> PQMF synthesis
                                                                       4096 streams x 2048
  cfg5  PQMF analysis 16 -> conv K7 16->64 -> 4 x [3 x residual(LReLU.2, conv K3 d=1,3,5),
        LReLU.2, strided conv K=2r+1 doubling] -> LReLU.2 -> conv K3 1024->256 (mean|var)
        -> slice mean 128 -> cfg4 decoder -> PQMF synthesis           16384 streams x
                                                                       {512, 2048, 8192}
All weights Kaiming-uniform from the seed (LeakyReLU(0.2) gain) with zero bias — the literal
BASELINE init for cfg1-cfg4.  cfg5 only [decision, evidenced]: its 27 residual-branch convs
(12 encoder + 15 decoder units) are additionally scaled by RES_SCALE_CFG5 = 0.5.  With plain
Kaiming the stacks compound to a pre-gate RMS of O(100), where the sigmoid gate turns
fp32-level relative errors into output errors above the 1e-4 x RMS tolerance for ANY
fp32-accumulating implementation: tests/test_oracle.py::test_res_scale_evidence runs the
oracle with an fp32-accumulating conv (oc_conv1d_f32acc) and asserts exactly that (cfg5 at
scale 1 fails the bound, at 0.5 passes; cfg4 at the literal init passes).  At 0.5 every layer
stays at RMS O(0.1-1) and the tolerance measures the kernels, not the model's conditioning.
`build(cfg, res_scale=...)` overrides the scale (the evidence test; cfg4 with 0.5 is the
round-1 variant).
Inputs are seeded synthetic (no dataset exists for this path; BASELINE.json names none).
"""
from __future__ import annotations

import math

import numpy as np

from .graph import Model

SR = 48000
RES_SCALE_CFG5 = 0.5

# frames = input frames per call per stream; out = output samples per call per stream
CONFIGS = {
    1: dict(name="cached_conv_64", streams=1, frames=2048, out=2048, buffers=64, in_channels=64),
    2: dict(name="residual_stack_c128", streams=256, frames=2048, out=2048, buffers=1,
            in_channels=128),
    3: dict(name="strided_encdec", streams=1024, frames=4096, out=4096, buffers=1, in_channels=16),
    4: dict(name="rave_decoder", streams=4096, frames=1, out=2048, buffers=1, in_channels=128),
    5: dict(name="rave_encdec", streams=16384, frames=2048, out=2048, buffers=1, in_channels=1),
}


def cfg1(seed: int = 0) -> Model:
    m = Model(64, seed)
    m.conv(64, 64, 3, padding="causal")
    return m


def cfg2(seed: int = 0) -> Model:
    m = Model(128, seed)
    for d in (1, 3, 9, 27):
        with m.residual():
            m.leaky_relu(0.2)
            m.conv(128, 128, 3, dilation=d, padding=(d, d))
            m.leaky_relu(0.2)
            m.conv(128, 128, 1, padding=(0, 0))
    return m


def cfg3(seed: int = 0, mirror: bool = True) -> Model:
    m = Model(16, seed)
    chans = [16, 64, 128, 256, 512]
    strides = [4, 4, 4, 2]
    for i, s in enumerate(strides):
        if i:
            m.leaky_relu(0.2)
        m.conv(chans[i], chans[i + 1], 2 * s + 1, stride=s, padding=(s, s))
    dec = strides[::-1] if mirror else strides
    rc = chans[::-1]
    for i, r in enumerate(dec):
        m.leaky_relu(0.2)
        m.conv_transpose(rc[i], rc[i + 1], 2 * r, r, padding=(r, r - 1))
    return m


def _decoder(m: Model, latent: int = 128, res_scale: float = 1.0) -> Model:
    m.conv(latent, 1024, 7, padding=(3, 3))
    c = 1024
    for r in (4, 4, 4, 2):
        m.leaky_relu(0.2)
        m.conv_transpose(c, c // 2, 2 * r, r, padding=(r, r - 1))
        c //= 2
        for d in (1, 3, 5):
            with m.residual():
                m.leaky_relu(0.2)
                m.conv(c, c, 3, dilation=d, padding=(d, d), scale=res_scale)
    m.leaky_relu(0.2)
    m.conv(c, 32, 7, padding=(3, 3))  # 16 wave + 16 amplitude channels
    m.gate()
    m.pqmf_synthesis(16, 256)
    return m


def cfg4(seed: int = 0, res_scale: float = 1.0, pqmf_design=None) -> Model:
    return _decoder(Model(128, seed, pqmf_design=pqmf_design), res_scale=res_scale)


def cfg5(seed: int = 0, res_scale: float = RES_SCALE_CFG5, pqmf_design=None) -> Model:
    m = Model(1, seed, pqmf_design=pqmf_design)
    m.pqmf_analysis(16, 256)
    m.conv(16, 64, 7, padding=(3, 3))
    c = 64
    for r in (4, 4, 4, 2):
        for d in (1, 3, 5):
            with m.residual():
                m.leaky_relu(0.2)
                m.conv(c, c, 3, dilation=d, padding=(d, d), scale=res_scale)
        m.leaky_relu(0.2)
        m.conv(c, 2 * c, 2 * r + 1, stride=r, padding=(r, r))
        c *= 2
    m.leaky_relu(0.2)
    m.conv(1024, 256, 3, padding=(1, 1))  # mean | variance (variance computed, dropped)
    m.slice(0, 128)
    return _decoder(m, 128, res_scale=res_scale)


BUILDERS = {1: cfg1, 2: cfg2, 3: cfg3, 4: cfg4, 5: cfg5}


def build(cfg: int, seed: int = 0, res_scale: float | None = None, pqmf_design=None) -> Model:
    """Config `cfg` with weights from `seed`.  pqmf_design: (bands, taps) -> (analysis,
    synthesis) for the PQMF stages (None: the library's sc_pqmf_filters; the oracle side passes
    oracle.pqmf_design.filters).  res_scale: override the residual-branch scale (cfg4/cfg5)."""
    if cfg in (4, 5):
        kw = dict(pqmf_design=pqmf_design)
        if res_scale is not None:
            kw["res_scale"] = res_scale
        return BUILDERS[cfg](seed, **kw)
    return BUILDERS[cfg](seed)


# ----------------------------------------------------------------------------- inputs
def stream_input(cfg: int, stream: int, channels: int, length: int, seed: int = 0) -> np.ndarray:
    """[channels][length] fp32 input of GLOBAL stream index `stream` (shard-independent)."""
    rng = np.random.default_rng([seed, 7919, stream])
    if cfg != 5:
        return rng.standard_normal((channels, length), dtype=np.float32)
    return audio_input(rng, length)


def audio_input(rng: np.random.Generator, length: int) -> np.ndarray:
    """cfg5: band-limited pink noise + random sine partials (f0 ~ U(55, 880) Hz, 8 harmonics,
    random decaying amplitudes), mono, peak-safe."""
    n = length
    spec = rng.standard_normal(n // 2 + 1) + 1j * rng.standard_normal(n // 2 + 1)
    f = np.fft.rfftfreq(n, 1.0 / SR)
    shape = np.zeros_like(f)
    band = (f >= 40.0) & (f <= 16000.0)
    shape[band] = 1.0 / np.sqrt(f[band])          # 1/f power = pink
    pink = np.fft.irfft(spec * shape, n)
    pink /= (np.sqrt(np.mean(pink ** 2)) + 1e-12)
    t = np.arange(n) / SR
    f0 = rng.uniform(55.0, 880.0)
    sig = 0.1 * pink
    for k in range(1, 9):
        if k * f0 >= SR / 2:
            break
        amp = rng.uniform(0.3, 1.0) * k ** -1.5 * 0.3
        decay = rng.uniform(0.5, 4.0)            # 1/s
        sig += amp * np.exp(-decay * t) * np.sin(2 * math.pi * k * f0 * t + rng.uniform(0, 2 * math.pi))
    return sig.astype(np.float32)[None, :]


def batch_input(cfg: int, streams, channels: int, length: int, seed: int = 0) -> np.ndarray:
    return np.stack([stream_input(cfg, s, channels, length, seed) for s in streams])

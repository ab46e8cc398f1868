"""Independent restatement of the PQMF filter-bank design (TEST INFRASTRUCTURE ONLY — used by
tests/, smoke() and bench.py's cpu_baseline / --impl reference legs; the product never imports
it).

The reference has no PQMF (it is named only in PAPER.md:114 as RAVE's
multiband decomposition), so the path's filter bank is pinned to the PUBLISHED algorithm
instead: the Kaiser-window approach to the prototype of a pseudo-QMF cosine-modulated filter
bank (Y.-P. Lin and P. P. Vaidyanathan, "A Kaiser window approach for the design of prototype
filters of cosine modulated filterbanks", IEEE Signal Processing Letters 5(6), 1998):

  prototype  p[n] = w_kaiser[n; beta] * sin(wc (n - (N-1)/2)) / (pi (n - (N-1)/2)),
             beta = 0.1102 (A - 8.7) for stop-band attenuation A = 100 dB (Kaiser's formula),
             wc   = argmin_wc  max_{m >= 1} | (p * p~)[2 M m] |   (the 2M-lag autocorrelation
             must vanish for near-perfect reconstruction — the paper's objective function);
  analysis   h_k[n] = 2 p[n] cos((2k+1) pi / (2M) (n - (N-1)/2) + (-1)^k pi/4)
  synthesis  f_k[n] = 2 p[n] cos((2k+1) pi / (2M) (n - (N-1)/2) - (-1)^k pi/4)
             (the standard cosine-modulation pair, e.g. Vaidyanathan, "Multirate Systems and
             Filter Banks", 1993, §8).

This module computes all of it in numpy double precision with its own primitives — the window
is `numpy.kaiser`, the sinc `numpy.sinc`, the autocorrelation `numpy.correlate`, the search a
dense grid followed by `scipy.optimize.minimize_scalar` (bounded Brent) around the best grid
point — so it shares no code with the product's `sc_pqmf_filters` (csrc/pqmf.cpp: hand-written
Bessel series + golden-section search).  tests/test_host.py pins the product's filters to this
design (max abs difference <= 1e-7), and the oracle-side models of cfg4 / cfg5 take their
PQMF weights from here.

Returned in the reference Kernel layout the runtime consumes (tensor.hpp:52-88, [n][m][k] +
bias[n], flat):
  analysis  CONV  (1 -> M, K = N, stride M, pad (N - M, 0)):  w[k][0][j] = h_k[N-1-j]
  synthesis CONVT (M -> 1, K = N, stride M, pad (N - 1, 0)):  w[0][k][j] = M f_k[N-1-j]
(conv1d is a correlation, kernels.cpp:96-98, so the convolution filters appear time-reversed;
the synthesis gain M undoes the M-fold decimation/upsampling energy loss).
"""
from __future__ import annotations

import functools

import numpy as np


def kaiser_beta(atten_db: float) -> float:
    """Kaiser's empirical beta for attenuation A > 50 dB."""
    return 0.1102 * (atten_db - 8.7)


def prototype(M: int, N: int, wc: float, beta: float) -> np.ndarray:
    t = np.arange(N, dtype=np.float64) - (N - 1) / 2.0
    ideal = (wc / np.pi) * np.sinc(wc * t / np.pi)      # sin(wc t) / (pi t)
    return ideal * np.kaiser(N, beta)


def objective(M: int, N: int, wc: float, beta: float) -> float:
    p = prototype(M, N, wc, beta)
    r = np.correlate(p, p, mode="full")[N - 1:]         # r[lag], lag = 0 .. N-1
    lags = np.arange(2 * M, N, 2 * M)
    return float(np.max(np.abs(r[lags]))) if lags.size else 0.0


@functools.lru_cache(maxsize=None)
def design(M: int = 16, N: int = 256, atten_db: float = 100.0):
    """(prototype p, cutoff wc) of the Kaiser-window PQMF prototype."""
    if M < 2 or N < 2 * M:
        raise ValueError("pqmf: need bands >= 2 and taps >= 2*bands")
    from scipy.optimize import minimize_scalar
    beta = kaiser_beta(atten_db)
    lo, hi = 0.5 * np.pi / (2 * M), 1.5 * np.pi / (2 * M)
    grid = np.linspace(lo, hi, 4001)
    vals = np.array([objective(M, N, w, beta) for w in grid])
    i = int(np.argmin(vals))
    a, b = grid[max(i - 1, 0)], grid[min(i + 1, grid.size - 1)]
    res = minimize_scalar(lambda w: objective(M, N, w, beta), bounds=(a, b), method="bounded",
                          options={"xatol": 1e-15, "maxiter": 500})
    wc = float(res.x)
    return prototype(M, N, wc, beta), wc


def cosine_modulated(M: int, N: int, p: np.ndarray):
    n = np.arange(N, dtype=np.float64)[None, :]
    k = np.arange(M, dtype=np.float64)[:, None]
    arg = (2 * k + 1) * np.pi / (2 * M) * (n - (N - 1) / 2.0)
    ph = np.where(np.arange(M) % 2 == 0, 1.0, -1.0)[:, None] * np.pi / 4
    h = 2.0 * p[None, :] * np.cos(arg + ph)
    f = 2.0 * p[None, :] * np.cos(arg - ph)
    return h, f


def filters(M: int = 16, N: int = 256):
    """(analysis, synthesis) flat fp32 weight arrays (+ zero biases), reference layout."""
    p, _ = design(M, N)
    h, f = cosine_modulated(M, N, p)
    ana = np.zeros(M * N + M, np.float32)
    syn = np.zeros(M * N + 1, np.float32)
    ana[:M * N] = h[:, ::-1].astype(np.float32).ravel()
    syn[:M * N] = (M * f[:, ::-1]).astype(np.float32).ravel()
    return ana, syn


def twin(model):
    """The oracle-side twin of an already built flat Model (paper_2204_07064_b200.graph.Model):
    a shallow copy whose PQMF stages (nodes hinted HINT_PQMF = 1, the analysis CONV and the
    synthesis CONVT) carry this module's filters instead of the product's sc_pqmf_filters.
    Models without PQMF stages come back unchanged (same object)."""
    import copy
    HINT_PQMF, NODE_CONV = 1, 0       # include/streamconv_b200.h: SC_HINT_PQMF, SC_NODE_CONV
    pq = [nd for nd in getattr(model, "nodes", []) if nd.get("hint") == HINT_PQMF]
    if not pq:
        return model
    tw = copy.copy(model)
    tw.chunks = list(model.chunks)
    starts = np.cumsum([0] + [c.size for c in model.chunks])[:-1].tolist()
    for nd in pq:
        i = starts.index(nd["weight_offset"])
        ana, syn = filters(max(nd["in_channels"], nd["out_channels"]), nd["taps"])
        new = ana if nd["kind"] == NODE_CONV else syn
        if new.size != tw.chunks[i].size:
            raise ValueError("PQMF stage shape does not match the design")
        tw.chunks[i] = new
    return tw

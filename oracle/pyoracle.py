"""ctypes front of the CPU ORACLE (test infrastructure only — tests/, smoke(), bench.py's
cpu_baseline and --impl reference legs).  The product package never imports this module.

  liboracle.so            oracle/oracle.cpp: restatement of kernels.cpp + SPEC stream_runtime
  libref_streamconv.so    the reference's own kernels.cpp (oracle/_ref, built by oracle/Makefile)
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "build" / "liboracle.so"
REF_SO = HERE / "_ref" / "libref_streamconv.so"

_o = None
_r = None

F32P = C.POINTER(C.c_float)
I64P = C.POINTER(C.c_int64)


def _fp(a: np.ndarray):
    return a.ctypes.data_as(F32P)


def oracle() -> C.CDLL:
    global _o
    if _o is None:
        if not ORACLE_SO.exists():
            raise RuntimeError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(str(ORACLE_SO))
        L.oc_last_error.restype = C.c_char_p
        L.oc_conv1d.argtypes = [F32P, C.c_int, C.c_int64, F32P, F32P, C.c_int, C.c_int, C.c_int,
                                C.c_int, F32P]
        L.oc_conv1d.restype = None
        L.oc_conv_output_length.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_int]
        L.oc_conv_output_length.restype = C.c_int64
        L.oc_delay_for_stride.argtypes = [C.c_int64, C.c_int64, C.c_int64]
        L.oc_delay_for_stride.restype = C.c_int64
        L.oc_branch_alignment.argtypes = [I64P, C.c_int, I64P]
        L.oc_pad_zeros.argtypes = [F32P, C.c_int, C.c_int64, C.c_int64, C.c_int64, F32P]
        L.oc_pad_zeros.restype = None
        L.oc_zero_upsample.argtypes = [F32P, C.c_int, C.c_int64, C.c_int, F32P]
        L.oc_zero_upsample.restype = None
        L.oc_activation.argtypes = [F32P, C.c_int64, C.c_int, C.c_float, F32P]
        L.oc_activation.restype = None
        L.oc_graph_info.argtypes = [C.c_void_p, C.c_int, F32P, C.c_int64, C.c_int, I64P]
        L.oc_dag_info.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, F32P, C.c_int64, C.c_int,
                                  I64P]
        L.oc_dag_run.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, F32P, C.c_int64, C.c_int,
                                 C.c_int, F32P, C.c_int64, I64P, C.c_int, F32P, C.c_int, C.c_void_p,
                                 C.c_int]
        L.oc_conv1d_f32acc.argtypes = L.oc_conv1d.argtypes
        L.oc_conv1d_f32acc.restype = None
        L.oc_set_f32acc_order.argtypes = [C.c_int]
        L.oc_run.argtypes = [C.c_void_p, C.c_int, F32P, C.c_int64, C.c_int, C.c_int, F32P,
                             C.c_int64, I64P, C.c_int, F32P, C.c_int, C.c_void_p, C.c_int]
        _o = L
    return _o


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> C.CDLL:
    global _r
    if _r is None:
        if not REF_SO.exists():
            raise RuntimeError(f"{REF_SO} missing (reference tree absent at build time)")
        L = C.CDLL(str(REF_SO))
        L.ref_conv1d.argtypes = [F32P, C.c_int, C.c_int64, F32P, F32P, C.c_int, C.c_int, C.c_int,
                                 C.c_int, F32P]
        L.ref_conv1d.restype = None
        L.ref_conv1d_checked.argtypes = [F32P, C.c_int, C.c_int64, F32P, F32P, C.c_int, C.c_int,
                                         C.c_int, C.c_int, F32P, C.c_int]
        L.ref_last_error.restype = C.c_char_p
        L.ref_pad_zeros.argtypes = [F32P, C.c_int, C.c_int64, C.c_int64, C.c_int64, F32P]
        L.ref_zero_upsample.argtypes = [F32P, C.c_int, C.c_int64, C.c_int, F32P]
        L.ref_activation.argtypes = [F32P, C.c_int64, C.c_int, C.c_float, F32P]
        L.ref_conv_output_length.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_int]
        L.ref_conv_output_length.restype = C.c_int64
        L.ref_set_parallel_kernels.argtypes = [C.c_int]
        _r = L
    return _r


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


# ----------------------------------------------------------------------- tensor_core
def conv1d(x: np.ndarray, w: np.ndarray, b: np.ndarray, stride: int = 1, dilation: int = 1,
           use_ref: bool = False) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    w = np.ascontiguousarray(w, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    M, L = x.shape
    N, M2, K = w.shape
    assert M == M2
    Lo = (L - ((K - 1) * dilation + 1)) // stride + 1
    y = np.zeros((N, max(Lo, 0)), np.float32)
    if use_ref:
        st = ref().ref_conv1d_checked(_fp(x), M, L, _fp(w), _fp(b), N, K, stride, dilation, _fp(y), 1)
        if st:
            raise OracleError(st, ref().ref_last_error().decode())
    else:
        oracle().oc_conv1d(_fp(x), M, L, _fp(w), _fp(b), N, K, stride, dilation, _fp(y))
    return y


def pad_zeros(x, left, right, use_ref=False):
    x = np.ascontiguousarray(x, np.float32)
    Cc, L = x.shape
    y = np.zeros((Cc, L + left + right), np.float32)
    if use_ref:
        ref().ref_pad_zeros(_fp(x), Cc, L, left, right, _fp(y))
    else:
        oracle().oc_pad_zeros(_fp(x), Cc, L, left, right, _fp(y))
    return y


def zero_upsample(x, factor, use_ref=False):
    x = np.ascontiguousarray(x, np.float32)
    Cc, L = x.shape
    y = np.zeros((Cc, L * factor), np.float32)
    if use_ref:
        ref().ref_zero_upsample(_fp(x), Cc, L, factor, _fp(y))
    else:
        oracle().oc_zero_upsample(_fp(x), Cc, L, factor, _fp(y))
    return y


def activation(x, kind, alpha=0.01, use_ref=False):
    x = np.ascontiguousarray(x, np.float32).ravel()
    y = np.zeros_like(x)
    (ref().ref_activation if use_ref else oracle().oc_activation)(_fp(x), x.size, kind, alpha, _fp(y))
    return y


def delay_for_stride(S, R, Dc):
    return oracle().oc_delay_for_stride(S, R, Dc)


def branch_alignment(D):
    d = np.ascontiguousarray(D, np.int64)
    a = np.zeros_like(d)
    st = oracle().oc_branch_alignment(d.ctypes.data_as(I64P), d.size, a.ctypes.data_as(I64P))
    if st:
        raise OracleError(st, "branch_alignment")
    return a.tolist()


# ----------------------------------------------------------------------- stream runtime
def _is_dag(model) -> bool:
    return hasattr(model, "edges")


def graph_info(model) -> dict:
    if _is_dag(model):
        nodes, n, edges, ne, w = model.pack()
        info = np.zeros(6, np.int64)
        st = oracle().oc_dag_info(C.cast(nodes, C.c_void_p), n, C.cast(edges, C.c_void_p), ne, _fp(w),
                                  w.size, model.in_channels, info.ctypes.data_as(I64P))
        if st:
            raise OracleError(st, oracle().oc_last_error().decode())
        return dict(ratio=int(info[0]), sink_num=int(info[1]), sink_den=int(info[2]),
                    out_channels=int(info[3]), latency_in=int(info[4]), state_bytes=int(info[5]))
    nodes, n, w = model.pack()
    info = np.zeros(6, np.int64)
    st = oracle().oc_graph_info(C.cast(nodes, C.c_void_p), n, _fp(w), w.size, model.in_channels,
                                info.ctypes.data_as(I64P))
    if st:
        raise OracleError(st, oracle().oc_last_error().decode())
    return dict(ratio=int(info[0]), sink_num=int(info[1]), sink_den=int(info[2]),
                out_channels=int(info[3]), latency_sink=int(info[4]), state_bytes=int(info[5]))


MODES = {"stream": 0, "offline": 1, "offline_original": 2, "phase": 3}


def _conv_ptr(use_ref, conv):
    if conv == "f32acc":        # evidence only: an fp32-accumulating conv (RES_SCALE test)
        return C.cast(oracle().oc_conv1d_f32acc, C.c_void_p)
    return C.cast(ref().ref_conv1d, C.c_void_p) if use_ref else None


def run(model, x: np.ndarray, parts=None, mode: str = "stream", use_ref: bool = False,
        threads: int = 0, conv: str | None = None) -> np.ndarray:
    """x: [streams][in_C][T].  Returns [streams][out_C][T*sink].  `model`: a flat Model or a
    SPEC DAG (graph.Graph, run by the oracle's independent DAG restatement).
    conv=None: the restatement (or the reference's conv1d when use_ref); "f32acc": the
    fp32-accumulating evidence conv (oc_conv1d_f32acc)."""
    if _is_dag(model):
        nodes, n, edges, ne, w = model.pack()
        x = np.ascontiguousarray(x, np.float32)
        S, Cin, T = x.shape
        info = graph_info(model)
        y = np.zeros((S, info["out_channels"], T * info["sink_num"] // info["sink_den"]), np.float32)
        p = np.ascontiguousarray([T] if parts is None else parts, np.int64)
        fn = _conv_ptr(use_ref, conv)
        st = oracle().oc_dag_run(C.cast(nodes, C.c_void_p), n, C.cast(edges, C.c_void_p), ne, _fp(w),
                                 w.size, model.in_channels, S, _fp(x), T, p.ctypes.data_as(I64P),
                                 p.size, _fp(y), MODES[mode], fn, threads)
        if st:
            raise OracleError(st, oracle().oc_last_error().decode())
        return y
    nodes, n, w = model.pack()
    x = np.ascontiguousarray(x, np.float32)
    S, Cin, T = x.shape
    info = graph_info(model)
    To = T * info["sink_num"] // info["sink_den"]
    y = np.zeros((S, info["out_channels"], To), np.float32)
    if parts is None:
        parts = [T]
    p = np.ascontiguousarray(parts, np.int64)
    fn = _conv_ptr(use_ref, conv)
    st = oracle().oc_run(C.cast(nodes, C.c_void_p), n, _fp(w), w.size, model.in_channels, S,
                         _fp(x), T, p.ctypes.data_as(I64P), p.size, _fp(y), MODES[mode], fn,
                         threads)
    if st:
        raise OracleError(st, oracle().oc_last_error().decode())
    return y


def host_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


# ----------------------------------------------------------------------- baseline_ola + metrics
def ola_window(n: int, overlap: int) -> np.ndarray:
    """SPEC hann_window: 50 -> sin^2(pi k / N); 25 -> the flat-top decision
    (sin^2 quarter lobes); 0 -> rectangular.  Double precision."""
    k = np.arange(n, dtype=np.float64)
    if overlap == 50:
        return np.sin(np.pi * k / n) ** 2
    w = np.ones(n)
    if overlap == 25:
        q = n // 4
        j = np.arange(q, dtype=np.float64)
        w[:q] = np.sin(np.pi * j / (2 * q)) ** 2
        w[n - q:] = np.sin(np.pi * (q - j) / (2 * q)) ** 2
    return w


def ola(model, x: np.ndarray, chunk: int, overlap: int) -> np.ndarray:
    """SPEC ola_process: chunks x[i*hop : i*hop+N] through offline_run of the
    ORIGINAL graph, times the ratio-scaled window, summed at offsets i*hop, trimmed to x."""
    S, Cin, T = x.shape
    hop = chunk * (100 - overlap) // 100
    nc = (T - chunk) // hop + 1
    chunks = np.stack([x[:, :, i * hop:i * hop + chunk] for i in range(nc)], axis=1)
    out = run(model, chunks.reshape(S * nc, Cin, chunk), mode="offline_original")
    No = out.shape[-1]
    out = out.reshape(S, nc, out.shape[1], No)
    hop_o = hop * No // chunk
    w = ola_window(No, overlap).astype(np.float32)
    y = np.zeros((S, out.shape[2], T * No // chunk), np.float32)
    for i in range(nc):
        y[:, :, i * hop_o:i * hop_o + No] += w * out[:, i]
    return y


def spectral_distance(x: np.ndarray, y: np.ndarray) -> float:
    """SPEC spectral_distance (Eq. 3 with epsilon 1): scales 256/512/1024, hop
    n/4, Hann sin^2 window, || log(|X|+1) - log(|Y|+1) ||_2 / frames, summed over scales."""
    x = np.asarray(x, np.float64).ravel()
    y = np.asarray(y, np.float64).ravel()
    if x.size != y.size:
        raise OracleError(14, "LengthMismatch")
    T = x.size
    total = 0.0
    for n in (256, 512, 1024):
        if T < n:
            continue
        hop = n // 4
        F = 1 + (T - n) // hop
        idx = np.arange(F)[:, None] * hop + np.arange(n)[None, :]
        w = np.sin(np.pi * np.arange(n) / n) ** 2
        X = np.abs(np.fft.rfft(x[idx] * w, axis=1))
        Y = np.abs(np.fft.rfft(y[idx] * w, axis=1))
        total += np.sqrt(np.sum((np.log1p(X) - np.log1p(Y)) ** 2)) / F
    return float(total)


def euclidean_distance(x, y) -> float:
    x = np.asarray(x, np.float64).ravel()
    y = np.asarray(y, np.float64).ravel()
    return float(np.sqrt(np.sum((x - y) ** 2)))


def correlation(x, y) -> float:
    x = np.asarray(x, np.float64).ravel()
    y = np.asarray(y, np.float64).ravel()
    ex, ey = np.sum(x * x), np.sum(y * y)
    if ex <= 0 or ey <= 0:
        raise OracleError(15, "ZeroEnergy")
    return float(np.sum(x * y) / np.sqrt(ex * ey))


def best_lag(ref, test, max_lag: int) -> int:
    ref = np.asarray(ref, np.float64).ravel()
    test = np.asarray(test, np.float64).ravel()
    T = ref.size
    best, bv = -1, -2.0
    for lag in range(max_lag + 1):
        a, b = ref[:T - lag], test[lag:]
        ea, eb = np.sum(a * a), np.sum(b * b)
        if ea <= 0 or eb <= 0:
            continue
        c = np.sum(a * b) / np.sqrt(ea * eb)
        if c > bv:
            best, bv = lag, c
    if best < 0:
        raise OracleError(15, "ZeroEnergy")
    return best

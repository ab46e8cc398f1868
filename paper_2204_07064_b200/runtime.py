"""Plan / StreamState: the Python face of the C-ABI (include/streamconv_b200.h).

Mirrors the reference stream_runtime: `Plan` = causalize(g) + device
weights, `StreamState` = init_state for a batch of independent streams, `.process_buffer` =
process_buffer for all of them in one asynchronous call, `.reset` = reset.  Errors raise
`StreamconvError` whose `.code` is the reference ErrCode name (error.hpp:8-29).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from ._abi import PREC_BF16, PREC_FP32, check, lib


def _stream_handle(stream) -> int:
    if stream is None:
        try:
            import torch
            return torch.cuda.current_stream().cuda_stream
        except Exception:  # pragma: no cover
            return 0
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


def _hptr(t) -> int:
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return int(t)


def _ptr(t) -> int:
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return int(t)


def _check_io(t, name: str, shape, dtypes, where: str, device: int = -1) -> None:
    """Validate a tensor / array handed to the C-ABI as a raw pointer: a wrong dtype, layout,
    device or size would otherwise become out-of-bounds device reads / writes.  Plain integer
    pointers are the caller's responsibility (raw C-ABI semantics)."""
    if isinstance(t, int):
        return
    shape = tuple(int(v) for v in shape)
    if isinstance(t, np.ndarray):
        if where != "host":
            raise ValueError(f"{name}: numpy arrays are host memory; a device tensor is required")
        if t.dtype.name not in dtypes:
            raise TypeError(f"{name}: dtype {t.dtype} not in {dtypes}")
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{name}: must be C-contiguous")
    elif hasattr(t, "data_ptr"):
        dt = str(t.dtype).replace("torch.", "")
        if dt not in dtypes:
            raise TypeError(f"{name}: dtype {t.dtype} not in {dtypes}")
        if not t.is_contiguous():
            raise ValueError(f"{name}: must be contiguous")
        if where == "device":
            if t.device.type != "cuda" or (device >= 0 and t.device.index != device):
                raise ValueError(f"{name}: must live on cuda:{device} (got {t.device})")
        elif t.device.type != "cpu":
            raise ValueError(f"{name}: must be a host (CPU) tensor (got {t.device})")
    else:
        raise TypeError(f"{name}: unsupported buffer type {type(t).__name__}")
    if tuple(t.shape) != shape:
        raise ValueError(f"{name}: shape {tuple(t.shape)} != expected {shape} "
                         "([n_streams][channels][frames])")


class Plan:
    def __init__(self, model, precision: str = "fp32", device: int = 0):
        """`model`: a flat cached-module stack (graph.Model) or a SPEC DAG (graph.Graph)."""
        from .graph import Graph
        prec = {"fp32": PREC_FP32, "bf16": PREC_BF16}[precision]
        h = C.c_void_p()
        self.in_channels = model.in_channels
        if isinstance(model, Graph):
            nodes, n, edges, ne, w = model.pack()
            self._w = w
            check(lib().sc_plan_create_graph(nodes, n, edges, ne,
                                             w.ctypes.data_as(C.POINTER(C.c_float)), w.size,
                                             model.in_channels, prec, device, C.byref(h)))
        else:
            nodes, n, w = model.pack()
            self._w = w
            check(lib().sc_plan_create(nodes, n, w.ctypes.data_as(C.POINTER(C.c_float)), w.size,
                                       model.in_channels, prec, device, C.byref(h)))
        self._h = h
        self.device = device
        self.precision = precision

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().sc_plan_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass

    @property
    def ratio(self) -> int:
        r = C.c_int64()
        check(lib().sc_plan_ratio(self._h, C.byref(r)))
        return r.value

    @property
    def sink(self):
        """(num, den, out_channels): output samples per input frame = num/den."""
        a, b, c = C.c_int64(), C.c_int64(), C.c_int32()
        check(lib().sc_plan_sink_rate(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    @property
    def latency(self) -> int:
        r = C.c_int64()
        check(lib().sc_plan_latency(self._h, C.byref(r)))
        return r.value

    @property
    def state_bytes(self) -> int:
        r = C.c_int64()
        check(lib().sc_plan_state_bytes(self._h, C.byref(r)))
        return r.value

    @property
    def macs_per_sample(self) -> float:
        r = C.c_double()
        check(lib().sc_plan_macs_per_sample(self._h, C.byref(r)))
        return r.value

    def op_macs(self):
        """Algorithmic MACs per stream per input sample of each fused op."""
        n = C.c_int32()
        check(lib().sc_plan_num_ops(self._h, C.byref(n)))
        out = []
        for i in range(n.value):
            v = C.c_double()
            check(lib().sc_plan_op_macs(self._h, i, C.byref(v)))
            out.append(v.value)
        return out

    def describe(self) -> str:
        return lib().sc_plan_describe(self._h).decode()

    def out_frames(self, frames: int) -> int:
        num, den, _ = self.sink
        return frames * num // den


class StreamState:
    def __init__(self, plan: Plan, n_streams: int, max_frames: int):
        self.plan = plan
        self.n_streams = n_streams
        self.max_frames = max_frames
        h = C.c_void_p()
        check(lib().sc_state_create(plan._h, n_streams, max_frames, C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().sc_state_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass

    def _io_shapes(self, frames: int):
        num, den, cout = self.plan.sink
        return ((self.n_streams, self.plan.in_channels, frames),
                (self.n_streams, cout, frames * num // den))

    def process_buffer(self, x, y, frames: int, stream=None) -> None:
        """x: device [n_streams][in_C][frames] fp32, y: device [n_streams][out_C][out_frames]."""
        si, so = self._io_shapes(frames)
        _check_io(x, "x", si, ("float32",), "device", self.plan.device)
        _check_io(y, "y", so, ("float32",), "device", self.plan.device)
        check(lib().sc_process(self._h, C.c_void_p(_ptr(x)), C.c_void_p(_ptr(y)), frames,
                               C.c_void_p(_stream_handle(stream))))

    def process_host(self, x, y, frames: int, stream=None) -> None:
        """Host-buffer process_buffer (pinned host memory for overlap): x/y host arrays or
        pinned torch CPU tensors with the same layouts as process_buffer."""
        si, so = self._io_shapes(frames)
        _check_io(x, "x", si, ("float32",), "host")
        _check_io(y, "y", so, ("float32",), "host")
        check(lib().sc_process_host(self._h, C.c_void_p(_hptr(x)), C.c_void_p(_hptr(y)), frames,
                                    C.c_void_p(_stream_handle(stream))))

    def process_host_bf16(self, x, y, frames: int, stream=None) -> None:
        """process_host with bf16 host buffers (torch.bfloat16 pinned tensors or uint16 arrays):
        half the PCIe bytes; outputs rounded to bf16 on the device."""
        si, so = self._io_shapes(frames)
        _check_io(x, "x", si, ("bfloat16", "uint16"), "host")
        _check_io(y, "y", so, ("bfloat16", "uint16"), "host")
        check(lib().sc_process_host_bf16(self._h, C.c_void_p(_hptr(x)), C.c_void_p(_hptr(y)), frames,
                                         C.c_void_p(_stream_handle(stream))))

    def host_wait(self, stream=None) -> None:
        """Order `stream` after the last process_host call's device->host copy."""
        check(lib().sc_process_host_wait(self._h, C.c_void_p(_stream_handle(stream))))

    def reset(self, stream_ids=None, stream=None) -> None:
        if stream_ids is None:
            check(lib().sc_state_reset(self._h, None, 0, C.c_void_p(_stream_handle(stream))))
        else:
            ids = np.ascontiguousarray(stream_ids, dtype=np.int32)
            check(lib().sc_state_reset(self._h, ids.ctypes.data_as(C.POINTER(C.c_int32)), ids.size,
                                       C.c_void_p(_stream_handle(stream))))

    def set_graphs(self, enabled: bool) -> None:
        check(lib().sc_state_set_graphs(self._h, 1 if enabled else 0))

    def launches(self, frames: int) -> int:
        n = C.c_int32()
        check(lib().sc_process_launches(self._h, frames, C.byref(n)))
        return n.value

    def launch_total(self) -> int:
        """Kernels this state has launched so far (sc_state_launch_total)."""
        n = C.c_int64()
        check(lib().sc_state_launch_total(self._h, C.byref(n)))
        return n.value

    def launch_names(self, frames: int):
        """Names of the launches one call of `frames` enqueues ("op<i> <op> [tc|tc-3xf16|tc-bf16|simt|pqmf]"; tc = 3xTF32, tc-3xf16 = 3xFP16)."""
        return [lib().sc_launch_name(self._h, frames, i).decode() for i in range(self.launches(frames))]

    def profile(self, x, y, frames: int, steps: int = 3, stream=None):
        """Per-launch mean device ms over `steps` un-graphed calls (CUDA events between
        launches on the launching stream).  Returns [(name, ms)]."""
        n = self.launches(frames)
        si, so = self._io_shapes(frames)
        _check_io(x, "x", si, ("float32",), "device", self.plan.device)
        _check_io(y, "y", so, ("float32",), "device", self.plan.device)
        ms = (C.c_float * n)()
        check(lib().sc_state_profile(self._h, C.c_void_p(_ptr(x)), C.c_void_p(_ptr(y)), frames,
                                     steps, ms, C.c_void_p(_stream_handle(stream))))
        return [(lib().sc_launch_name(self._h, frames, i).decode(), float(ms[i])) for i in range(n)]

    @property
    def device_bytes(self) -> int:
        r = C.c_int64()
        check(lib().sc_state_device_bytes(self._h, C.byref(r)))
        return r.value

    def redzone_violations(self) -> int:
        """Guard bytes overwritten since creation / full reset (-1: created without SC_REDZONE=1)."""
        r = C.c_int64()
        check(lib().sc_state_redzone_check(self._h, C.byref(r)))
        return r.value

    @property
    def cache_bytes(self) -> int:
        r = C.c_int64()
        check(lib().sc_state_cache_bytes(self._h, C.byref(r)))
        return r.value


class Ola:
    """SPEC baseline_ola on the GPU: overlap-add of the unmodified
    (non-causal) graph over windowed chunks, every chunk of every stream batched (sc_ola_*)."""

    def __init__(self, graph, chunk: int, overlap: int, n_streams: int, max_frames: int,
                 precision: str = "fp32", device: int = 0):
        from .graph import Graph, Model, model_to_graph
        if isinstance(graph, Model):
            graph = model_to_graph(graph)
        nodes, n, edges, ne, w = graph.pack()
        self._w = w
        self.chunk, self.overlap, self.n_streams = chunk, overlap, n_streams
        h = C.c_void_p()
        check(lib().sc_ola_create(nodes, n, edges, ne, w.ctypes.data_as(C.POINTER(C.c_float)), w.size,
                                  graph.in_channels, {"fp32": PREC_FP32, "bf16": PREC_BF16}[precision],
                                  device, chunk, overlap, n_streams, max_frames, C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                lib().sc_ola_destroy(self._h)
                self._h = None
        except Exception:  # interpreter shutdown
            pass

    def process(self, x, y, frames: int, stream=None) -> None:
        """x: device [n_streams][in_C][frames], y: device [n_streams][out_C][frames x sink]."""
        check(lib().sc_ola_process(self._h, C.c_void_p(_ptr(x)), C.c_void_p(_ptr(y)), frames,
                                   C.c_void_p(_stream_handle(stream))))

    def describe(self) -> str:
        return lib().sc_ola_describe(self._h).decode()

    @staticmethod
    def window(n: int, overlap: int) -> np.ndarray:
        w = np.zeros(n, np.float32)
        check(lib().sc_ola_window(n, overlap, w.ctypes.data_as(C.POINTER(C.c_float))))
        return w

    @staticmethod
    def redundancy(overlap: int) -> float:
        return lib().sc_ola_redundancy(overlap)


def fidelity(ref, test, stream=None):
    """SPEC metrics_bench scores of device signals [n][T] (or [n][1][T]): dict of numpy arrays
    L_s (spectral, Eq. 3), L_w (Euclidean, Eq. 4), L_c (correlation)."""
    n = int(ref.shape[0])
    T = int(ref.shape[-1])
    ls, lw, lc = (np.zeros(n, np.float64) for _ in range(3))
    dp = C.POINTER(C.c_double)
    check(lib().sc_fidelity(C.c_void_p(_ptr(ref)), C.c_void_p(_ptr(test)), n, T, ls.ctypes.data_as(dp),
                            lw.ctypes.data_as(dp), lc.ctypes.data_as(dp), C.c_void_p(_stream_handle(stream))))
    return dict(L_s=ls, L_w=lw, L_c=lc)


def best_lag(ref, test, max_lag: int, stream=None) -> np.ndarray:
    """SPEC best_lag per signal of device batches [n][T]."""
    n = int(ref.shape[0])
    out = np.zeros(n, np.int64)
    check(lib().sc_best_lag(C.c_void_p(_ptr(ref)), C.c_void_p(_ptr(test)), n, int(ref.shape[-1]), max_lag,
                            out.ctypes.data_as(C.POINTER(C.c_int64)), C.c_void_p(_stream_handle(stream))))
    return out


def conv1d(x, w, b, y, batch: int, in_channels: int, length: int, out_channels: int, taps: int,
           stride: int = 1, dilation: int = 1, stream=None) -> None:
    """Device conv1d (kernels.cpp:73-104) over a batch; reference layouts, device pointers."""
    check(lib().sc_conv1d(C.c_void_p(_ptr(x)), batch, in_channels, length, C.c_void_p(_ptr(w)),
                          C.c_void_p(_ptr(b)), out_channels, taps, stride, dilation,
                          C.c_void_p(_ptr(y)), C.c_void_p(_stream_handle(stream))))


def conv_output_length(length: int, taps: int, stride: int = 1, dilation: int = 1) -> int:
    return lib().sc_conv_output_length(length, taps, stride, dilation)


def delay_for_stride(stride: int, right_pad: int, cumulated: int) -> int:
    return lib().sc_delay_for_stride(stride, right_pad, cumulated)


def branch_alignment(delays):
    d = np.ascontiguousarray(delays, dtype=np.int64)
    out = np.zeros_like(d)
    check(lib().sc_branch_alignment(d.ctypes.data_as(C.POINTER(C.c_int64)), d.size,
                                    out.ctypes.data_as(C.POINTER(C.c_int64))))
    return out.tolist()

"""Cached-module API (Python mirror of csrc/modules.hpp): build a causalizable model as the
flat node list of the C-ABI (include/streamconv_b200.h, `sc_node`).

Vocabulary follows the reference (SPEC.md graph_ir) and the north star's
cached modules: cached Conv1d, cached ConvTranspose1d (SPEC's zero_upsample + conv,
SPEC.md:57-58,91), residual branches with delay alignment (Fanout/Sum), a
sequential stack, PQMF analysis/synthesis.  Paddings are given as the ORIGINAL (possibly
centered, non-causal) PaddingSpec{left,right} (tensor.hpp:90-95); the plan runs causalize.

Weights are in the reference Kernel layout [n][m][k] + bias[n] (tensor.hpp:52-88).
"""
from __future__ import annotations

import contextlib
import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._abi import (ACT_IDENTITY, ACT_LEAKY_RELU, ACT_TANH, NODE_ACT, NODE_CONV, NODE_CONVT,
                   NODE_GATE, NODE_RES_BEGIN, NODE_RES_END, NODE_SLICE, SCNode)

LRELU_GAIN = math.sqrt(2.0 / (1.0 + 0.2 ** 2))


def kaiming_uniform(rng: np.random.Generator, cout: int, cin: int, k: int, fan_in: float,
                    gain: float = LRELU_GAIN) -> np.ndarray:
    """U(-b, b), b = gain * sqrt(3 / fan_in): keeps signal RMS O(1) so RMS-relative tolerances
    are meaningful (SURVEY.md §7 [decision]; SPEC's synthetic init is U[-1/(MK), 1/(MK)],
    SPEC.md:452)."""
    b = gain * math.sqrt(3.0 / fan_in)
    return rng.uniform(-b, b, size=(cout, cin, k)).astype(np.float32)


@dataclass
class Model:
    """A sequential stack of cached modules (the node list of one causalizable graph)."""

    in_channels: int
    seed: int = 0
    nodes: list = field(default_factory=list)
    chunks: list = field(default_factory=list)
    _n_weights: int = 0
    _C: int = -1

    def __post_init__(self):
        self._rng = np.random.default_rng(self.seed)
        self._C = self.in_channels

    @property
    def channels(self) -> int:
        return self._C

    def _add_weights(self, w: np.ndarray, b: np.ndarray) -> int:
        off = self._n_weights
        flat = np.concatenate([np.ascontiguousarray(w, np.float32).ravel(),
                               np.ascontiguousarray(b, np.float32).ravel()])
        self.chunks.append(flat)
        self._n_weights += flat.size
        return off

    def _node(self, kind, **kw) -> dict:
        nd = dict(kind=kind, in_channels=0, out_channels=0, taps=0, stride=1, dilation=1,
                  pad_left=0, pad_right=0, act=0, alpha=0.0, weight_offset=0, slice_begin=0,
                  slice_count=0, hint=0)
        nd.update(kw)
        self.nodes.append(nd)
        return nd

    # ---- cached Conv1d: conv1d(pad(x,(L,R)), k, stride, dilation) (kernels.cpp:73-104)
    def conv(self, cin: int, cout: int, k: int, stride: int = 1, dilation: int = 1,
             padding=None, weight=None, bias=None, scale: float = 1.0) -> "Model":
        if padding is None or padding == "centered":
            tot = (k - 1) * dilation if stride == 1 else k - 1
            padding = ((tot + 1) // 2, tot // 2)
        elif padding == "causal":
            padding = ((k - 1) * dilation if stride == 1 else k - 1, 0)
        if weight is None:
            weight = kaiming_uniform(self._rng, cout, cin, k, cin * k) * np.float32(scale)
        if bias is None:
            bias = np.zeros(cout, np.float32)
        off = self._add_weights(weight, bias)
        self._node(NODE_CONV, in_channels=cin, out_channels=cout, taps=k, stride=stride,
                   dilation=dilation, pad_left=padding[0], pad_right=padding[1], weight_offset=off)
        self._C = cout
        return self

    # ---- cached ConvTranspose1d = zero_upsample(stride) + conv1d
    def conv_transpose(self, cin: int, cout: int, k: int, stride: int, padding=None,
                       weight=None, bias=None) -> "Model":
        if padding is None or padding == "centered":
            padding = ((k - 1 + 1) // 2, (k - 1) // 2)
        elif padding == "causal":
            padding = (k - 1, 0)
        if weight is None:
            weight = kaiming_uniform(self._rng, cout, cin, k, cin * k / stride)
        if bias is None:
            bias = np.zeros(cout, np.float32)
        off = self._add_weights(weight, bias)
        self._node(NODE_CONVT, in_channels=cin, out_channels=cout, taps=k, stride=stride,
                   dilation=1, pad_left=padding[0], pad_right=padding[1], weight_offset=off)
        self._C = cout
        return self

    # ---- activation (kernels.cpp:119-128); the reference default alpha is 0.01 (kernels.hpp:32)
    def act(self, kind: int, alpha: float = 0.01) -> "Model":
        self._node(NODE_ACT, act=kind, alpha=alpha)
        return self

    def leaky_relu(self, alpha: float = 0.01) -> "Model":
        return self.act(ACT_LEAKY_RELU, alpha)

    def tanh(self) -> "Model":
        return self.act(ACT_TANH)

    @contextlib.contextmanager
    def residual(self):
        """Fanout -> branch -> Sum(branch, Delay_A(skip)); A from branch_alignment."""
        c0 = self._C
        self._node(NODE_RES_BEGIN)
        yield self
        if self._C != c0:
            raise ValueError("residual branch must preserve channels")
        self._node(NODE_RES_END)

    def gate(self) -> "Model":
        """y[c] = tanh(x[c]) * sigmoid(x[c + C/2]) (RAVE amplitude-gated head; builder-defined)."""
        self._node(NODE_GATE)
        self._C //= 2
        return self

    def slice(self, begin: int, count: int) -> "Model":
        self._node(NODE_SLICE, slice_begin=begin, slice_count=count)
        self._C = count
        return self

    # ---- PQMF (builder-defined; parity unpinned): filters from sc_pqmf_filters
    def pqmf_analysis(self, bands: int = 16, taps: int = 256) -> "Model":
        ana, _ = pqmf_filters(bands, taps)
        w = ana[: bands * taps].reshape(bands, 1, taps)
        self.conv(1, bands, taps, stride=bands, padding=(taps - bands, 0), weight=w,
                  bias=np.zeros(bands, np.float32))
        self.nodes[-1]["hint"] = _abi.HINT_PQMF
        return self

    def pqmf_synthesis(self, bands: int = 16, taps: int = 256) -> "Model":
        _, syn = pqmf_filters(bands, taps)
        w = syn[: bands * taps].reshape(1, bands, taps)
        self.conv_transpose(bands, 1, taps, stride=bands, padding=(taps - 1, 0), weight=w,
                            bias=np.zeros(1, np.float32))
        self.nodes[-1]["hint"] = _abi.HINT_PQMF
        return self

    # ---- C-ABI form
    def pack(self):
        arr = (SCNode * max(1, len(self.nodes)))()
        for i, nd in enumerate(self.nodes):
            for kk, vv in nd.items():
                setattr(arr[i], kk, vv)
        w = (np.concatenate(self.chunks) if self.chunks else np.zeros(1, np.float32)).astype(np.float32)
        return arr, len(self.nodes), np.ascontiguousarray(w)


_PQMF_CACHE: dict = {}


def pqmf_filters(bands: int, taps: int):
    """Analysis/synthesis weights (+ zero biases) from the library's double-precision design."""
    key = (bands, taps)
    if key not in _PQMF_CACHE:
        import ctypes as C
        ana = np.zeros(bands * taps + bands, np.float32)
        syn = np.zeros(bands * taps + 1, np.float32)
        proto = np.zeros(taps, np.float64)
        _abi.check(_abi.lib().sc_pqmf_filters(
            bands, taps, ana.ctypes.data_as(C.POINTER(C.c_float)),
            syn.ctypes.data_as(C.POINTER(C.c_float)), proto.ctypes.data_as(C.POINTER(C.c_double))))
        _PQMF_CACHE[key] = (ana, syn, proto)
    ana, syn, _ = _PQMF_CACHE[key]
    return ana, syn


def pqmf_prototype(bands: int, taps: int) -> np.ndarray:
    pqmf_filters(bands, taps)
    return _PQMF_CACHE[(bands, taps)][2]

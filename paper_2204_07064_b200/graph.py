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
    # (bands, taps) -> (analysis, synthesis) flat weights; None = the library's own design
    # (sc_pqmf_filters).  The oracle side passes oracle.pqmf_design.filters, so a reference
    # run never loads the product library (bench.py --impl reference) and the parity tests
    # check the product's filter design against an independent one.
    pqmf_design: object = None

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
        ana, _ = (self.pqmf_design or pqmf_filters)(bands, taps)
        w = ana[: bands * taps].reshape(bands, 1, taps)
        self.conv(1, bands, taps, stride=bands, padding=(taps - bands, 0), weight=w,
                  bias=np.zeros(bands, np.float32))
        self.nodes[-1]["hint"] = _abi.HINT_PQMF
        return self

    def pqmf_synthesis(self, bands: int = 16, taps: int = 256) -> "Model":
        _, syn = (self.pqmf_design or pqmf_filters)(bands, taps)
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


class Graph:
    """SPEC graph_ir DAG: typed nodes joined by (from, to, port) edges.

    Builder methods take the producing node id(s) and return the new node's id; a node whose
    output feeds several consumers gets a Fanout of that arity inserted when the graph is
    packed (SPEC houses branching in Fanout nodes).  Weights use the reference Kernel layout
    ([n][m][k] + bias[n], tensor.hpp:52-88) in one flat array, like `Model`.
    """

    def __init__(self, in_channels: int, seed: int = 0):
        self.in_channels = in_channels
        self.nodes: list = []
        self.edges: list = []       # (from, to, port)
        self.chunks: list = []
        self._n_weights = 0
        self._rng = np.random.default_rng(seed)
        self.source = self.add(_abi.G_SOURCE, out_channels=in_channels)

    # ---- raw construction
    def add(self, kind: int, inputs=(), **kw) -> int:
        nd = dict(kind=kind, in_channels=0, out_channels=0, taps=0, stride=1, dilation=1,
                  pad_left=0, pad_right=0, shift=0, factor=1, act=0, alpha=0.0, arity=0,
                  samples=0, weight_offset=0, slice_begin=0, slice_count=0, hint=0, inserted=0)
        nd.update(kw)
        self.nodes.append(nd)
        i = len(self.nodes) - 1
        for port, src in enumerate(inputs):
            self.edges.append((src, i, port))
        return i

    def _add_weights(self, w: np.ndarray, b: np.ndarray) -> int:
        off = self._n_weights
        flat = np.concatenate([np.ascontiguousarray(w, np.float32).ravel(),
                               np.ascontiguousarray(b, np.float32).ravel()])
        self.chunks.append(flat)
        self._n_weights += flat.size
        return off

    # ---- SPEC NodeKinds
    def conv(self, x: int, cin: int, cout: int, k: int, stride: int = 1, dilation: int = 1,
             padding=None, weight=None, bias=None, init: str = "kaiming", hint: int = 0) -> int:
        """Conv{kernel, stride, dilation, padding} (kernels.cpp:73-104)."""
        if padding is None or padding == "centered":
            tot = (k - 1) * dilation if stride == 1 else k - 1
            padding = ((tot + 1) // 2, tot // 2)
        elif padding == "causal":
            padding = ((k - 1) * dilation if stride == 1 else k - 1, 0)
        if weight is None:
            if init == "spec":  # SPEC synthetic init U[-1/(MK), 1/(MK)]
                b_ = 1.0 / (cin * k)
                weight = self._rng.uniform(-b_, b_, size=(cout, cin, k)).astype(np.float32)
            else:
                weight = kaiming_uniform(self._rng, cout, cin, k, cin * k)
        if bias is None:
            bias = np.zeros(cout, np.float32)
        off = self._add_weights(weight, bias)
        return self.add(_abi.G_CONV, [x], in_channels=cin, out_channels=cout, taps=k,
                        stride=stride, dilation=dilation, pad_left=padding[0],
                        pad_right=padding[1], weight_offset=off, hint=hint)

    def zero_upsample(self, x: int, factor: int) -> int:
        return self.add(_abi.G_ZERO_UPSAMPLE, [x], factor=factor)

    def act(self, x: int, kind: int, alpha: float = 0.01) -> int:
        return self.add(_abi.G_ACTIVATION, [x], act=kind, alpha=alpha)

    def leaky_relu(self, x: int, alpha: float = 0.01) -> int:
        return self.act(x, ACT_LEAKY_RELU, alpha)

    def tanh(self, x: int) -> int:
        return self.act(x, ACT_TANH)

    def delay(self, x: int, samples: int) -> int:
        return self.add(_abi.G_DELAY, [x], samples=samples)

    def sum(self, *xs: int) -> int:
        return self.add(_abi.G_SUM, list(xs), arity=len(xs))

    def gate(self, x: int) -> int:
        return self.add(_abi.G_GATE, [x])

    def slice(self, x: int, begin: int, count: int) -> int:
        return self.add(_abi.G_SLICE, [x], slice_begin=begin, slice_count=count)

    def sink(self, x: int) -> int:
        return self.add(_abi.G_SINK, [x])

    # ---- C-ABI form
    def finalized(self) -> "Graph":
        """Copy with a Fanout inserted wherever a non-Fanout node feeds several consumers."""
        g = Graph.__new__(Graph)
        g.in_channels, g.chunks, g._n_weights, g._rng = (self.in_channels, self.chunks,
                                                          self._n_weights, self._rng)
        g.source = self.source
        g.nodes = [dict(nd) for nd in self.nodes]
        uses: dict = {}
        for e in self.edges:
            uses.setdefault(e[0], []).append(e)
        edges = []
        fan: dict = {}
        for i, nd in enumerate(self.nodes):
            us = uses.get(i, [])
            if len(us) > 1 and nd["kind"] != _abi.G_FANOUT:
                g.nodes.append(dict(kind=_abi.G_FANOUT, in_channels=0, out_channels=0, taps=0,
                                    stride=1, dilation=1, pad_left=0, pad_right=0, shift=0,
                                    factor=1, act=0, alpha=0.0, arity=len(us), samples=0,
                                    weight_offset=0, slice_begin=0, slice_count=0, hint=0,
                                    inserted=0))
                fan[i] = len(g.nodes) - 1
        for (a, b, p) in self.edges:  # edge order kept (Sum operand order)
            edges.append((fan.get(a, a), b, p))
        for a, f in fan.items():
            edges.append((a, f, 0))
        g.edges = edges
        return g

    def pack(self):
        g = self.finalized()
        nodes = (_abi.SCGNode * max(1, len(g.nodes)))()
        for i, nd in enumerate(g.nodes):
            for kk, vv in nd.items():
                setattr(nodes[i], kk, vv)
        edges = (_abi.SCEdge * max(1, len(g.edges)))()
        for i, (a, b, p) in enumerate(g.edges):
            edges[i].from_, edges[i].to, edges[i].port = a, b, p
        w = (np.concatenate(self.chunks) if self.chunks else np.zeros(1, np.float32)).astype(np.float32)
        return nodes, len(g.nodes), edges, len(g.edges), np.ascontiguousarray(w)

    @classmethod
    def from_arrays(cls, nodes, n_nodes: int, edges, n_edges: int, weights: np.ndarray,
                    in_channels: int) -> "Graph":
        g = cls.__new__(cls)
        g.in_channels = in_channels
        g._rng = np.random.default_rng(0)
        g.nodes = [{f: getattr(nodes[i], f) for f, _ in _abi.SCGNode._fields_} for i in range(n_nodes)]
        g.edges = [(edges[i].from_, edges[i].to, edges[i].port) for i in range(n_edges)]
        w = np.ascontiguousarray(weights, np.float32).copy()
        g.chunks = [w]
        g._n_weights = w.size
        g.source = next(i for i, nd in enumerate(g.nodes) if nd["kind"] == _abi.G_SOURCE)
        return g

    # ---- SPEC analyses (through the C-ABI)
    def _args(self):
        nodes, n, edges, ne, _ = self.pack()
        return nodes, n, edges, ne, self.in_channels

    def validate(self) -> dict:
        """SPEC validate: out channels and the RateMap of the packed edges."""
        import ctypes as C
        nodes, n, edges, ne, ic = self._args()
        rates = np.zeros((max(ne, 1), 2), np.int64)
        oc = C.c_int32()
        _abi.check(_abi.lib().sc_graph_validate(nodes, n, edges, ne, ic,
                                                rates.ctypes.data_as(C.POINTER(C.c_int64)),
                                                C.byref(oc)))
        return dict(out_channels=oc.value, rates=[tuple(r) for r in rates[:ne]])

    def compression_ratio(self) -> int:
        import ctypes as C
        r = C.c_int64()
        _abi.check(_abi.lib().sc_graph_compression_ratio(*self._args(), C.byref(r)))
        return r.value

    def receptive_field(self):
        import ctypes as C
        p, f = C.c_int64(), C.c_int64()
        _abi.check(_abi.lib().sc_graph_receptive_field(*self._args(), C.byref(p), C.byref(f)))
        return p.value, f.value

    def mac_count(self, input_samples: int) -> int:
        """SPEC mac_count: the literal offline MACs over input_samples."""
        import ctypes as C
        r = C.c_int64()
        _abi.check(_abi.lib().sc_graph_mac_count(*self._args(), input_samples, C.byref(r)))
        return r.value

    def latency(self) -> int:
        """SPEC latency_of; NotCausal for a graph with future context."""
        import ctypes as C
        r = C.c_int64()
        _abi.check(_abi.lib().sc_graph_latency(*self._args(), C.byref(r)))
        return r.value

    def causalize(self):
        """SPEC causalize: (causalized Graph, total latency in samples)."""
        import ctypes as C
        nodes, n, edges, ne, ic = self._args()
        cap_n, cap_e = n + ne, 2 * ne
        on = (_abi.SCGNode * cap_n)()
        oe = (_abi.SCEdge * max(cap_e, 1))()
        nn, nne, lat = C.c_int32(), C.c_int32(), C.c_int64()
        _abi.check(_abi.lib().sc_graph_causalize(nodes, n, edges, ne, ic, on, cap_n, C.byref(nn),
                                                 oe, cap_e, C.byref(nne), C.byref(lat)))
        w = np.concatenate(self.chunks) if self.chunks else np.zeros(1, np.float32)
        return Graph.from_arrays(on, nn.value, oe, nne.value, w, ic), lat.value

    # ---- SPEC model_io
    def save(self, manifest_path, blob_path=None) -> None:
        nodes, n, edges, ne, w = self.pack()
        _abi.check(_abi.lib().sc_model_save(
            str(manifest_path).encode(), None if blob_path is None else str(blob_path).encode(),
            nodes, n, edges, ne, w.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_float)),
            w.size, self.in_channels))

    @classmethod
    def load(cls, manifest_path, blob_path=None) -> "Graph":
        import ctypes as C
        h = C.c_void_p()
        _abi.check(_abi.lib().sc_model_load(str(manifest_path).encode(),
                                            None if blob_path is None else str(blob_path).encode(),
                                            C.byref(h)))
        try:
            pn, pe, pw = C.POINTER(_abi.SCGNode)(), C.POINTER(_abi.SCEdge)(), C.POINTER(C.c_float)()
            n, ne, nw, ic = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int32()
            _abi.check(_abi.lib().sc_model_graph(h, C.byref(pn), C.byref(n), C.byref(pe), C.byref(ne),
                                                 C.byref(pw), C.byref(nw), C.byref(ic)))
            w = np.ctypeslib.as_array(pw, shape=(nw.value,)).copy() if nw.value else np.zeros(1, np.float32)
            return cls.from_arrays(pn, n.value, pe, ne.value, w, ic.value)
        finally:
            _abi.lib().sc_model_destroy(h)


def model_to_graph(model: "Model") -> Graph:
    """The flat cached-module stack as a SPEC DAG: RES_BEGIN -> Fanout, RES_END ->
    Sum(branch, skip) in that operand order (the oracle's `br + skip`)."""
    g = Graph(model.in_channels)
    g.chunks = list(model.chunks)
    g._n_weights = model._n_weights
    x = g.source
    stack = []
    for nd in model.nodes:
        k = nd["kind"]
        if k in (NODE_CONV, NODE_CONVT):
            if k == NODE_CONVT:
                x = g.zero_upsample(x, nd["stride"])
            x = g.add(_abi.G_CONV, [x], in_channels=nd["in_channels"], out_channels=nd["out_channels"],
                      taps=nd["taps"], stride=1 if k == NODE_CONVT else nd["stride"],
                      dilation=nd["dilation"], pad_left=nd["pad_left"], pad_right=nd["pad_right"],
                      weight_offset=nd["weight_offset"], hint=nd["hint"])
        elif k == NODE_ACT:
            x = g.act(x, nd["act"], nd["alpha"])
        elif k == NODE_GATE:
            x = g.gate(x)
        elif k == NODE_SLICE:
            x = g.slice(x, nd["slice_begin"], nd["slice_count"])
        elif k == NODE_RES_BEGIN:
            stack.append(x)
        elif k == NODE_RES_END:
            x = g.sum(x, stack.pop())
    g.sink(x)
    return g


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


@dataclass
class SynthConfig:
    """SPEC SynthConfig: a deterministic RAVE-like model for tests/benchmarks."""

    strides: tuple = (4, 4, 2)
    base_channels: int = 8
    encoder_kernels: tuple = ()     # default 2*s+1 per stage
    res_blocks: int = 1             # residual blocks per decoder stage
    res_kernel: int = 3
    padding: str = "centered"       # "centered" | "causal"
    seed: int = 0
    in_channels: int = 1
    alpha: float = 0.2


def make_synthetic_rave(cfg: SynthConfig = SynthConfig()) -> Graph:
    """SPEC make_synthetic_rave: encoder Conv stack (the given strides, tanh
    between) -> decoder per stage: ZeroUpsample + Conv + residual blocks (Fanout ->
    [Conv-act-Conv, identity] -> Sum) -> Conv to the input channels.  Weights uniform in
    [-1/(M K), 1/(M K)] from the seed; centered padding gives a non-causal model (future > 0),
    causal padding a causal one."""
    if any(s < 1 for s in cfg.strides):
        raise ValueError("strides must be >= 1")
    if cfg.padding not in ("centered", "causal"):
        raise ValueError("padding must be 'centered' or 'causal'")
    g = Graph(cfg.in_channels, seed=cfg.seed)
    kern = list(cfg.encoder_kernels) or [2 * s + 1 for s in cfg.strides]
    chans = [cfg.base_channels * (2 ** i) for i in range(len(cfg.strides) + 1)]
    x = g.conv(g.source, cfg.in_channels, chans[0], 3, padding=cfg.padding, init="spec")
    for i, s in enumerate(cfg.strides):
        x = g.tanh(x)
        x = g.conv(x, chans[i], chans[i + 1], kern[i], stride=s, padding=cfg.padding, init="spec")
    for i in reversed(range(len(cfg.strides))):
        s = cfg.strides[i]
        x = g.leaky_relu(x, cfg.alpha)
        if s > 1:
            x = g.zero_upsample(x, s)
        k = 2 * s
        pad = (k - 1, 0) if cfg.padding == "causal" else (k // 2, k // 2 - 1)
        x = g.conv(x, chans[i + 1], chans[i], k, padding=pad, init="spec")
        for _ in range(cfg.res_blocks):
            h = g.leaky_relu(x, cfg.alpha)
            h = g.conv(h, chans[i], chans[i], cfg.res_kernel, padding=cfg.padding, init="spec")
            h = g.leaky_relu(h, cfg.alpha)
            h = g.conv(h, chans[i], chans[i], 1, padding=(0, 0), init="spec")
            x = g.sum(h, x)
    x = g.tanh(x)
    x = g.conv(x, chans[0], cfg.in_channels, 3, padding=cfg.padding, init="spec")
    g.sink(x)
    return g

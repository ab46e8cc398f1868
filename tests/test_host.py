"""CPU: the C-ABI library loads and exports every symbol include/*.h declares; host-only
plans (device -1: validation + causalize + lowering, no GPU) agree with the oracle's
causalize; typed errors cross the boundary as the reference ErrCodes (error.hpp:8-29)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2204_07064_b200 import StreamconvError, configs, lib
from paper_2204_07064_b200._abi import EXPORTED, SCNode
from paper_2204_07064_b200.graph import Model
from paper_2204_07064_b200.runtime import Plan, branch_alignment, conv_output_length, delay_for_stride

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    syms = set()
    for h in (ROOT / "include").glob("*.h"):
        for m in re.finditer(r"SC_API\s+[\w\s\*]+?\b(sc_\w+)\s*\(", h.read_text()):
            syms.add(m.group(1))
    return syms


def test_library_exports_every_declared_symbol():
    L = lib()
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert syms <= set(EXPORTED) | {"sc_version"}, syms - set(EXPORTED)
    assert b"sm_100a" in L.sc_version()


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_host_plan_matches_oracle_causalize(cfg):
    m = configs.build(cfg, seed=0)
    p = Plan(m, device=-1)
    o = po.graph_info(m)
    num, den, cout = p.sink
    assert (p.ratio, num, den, cout) == (o["ratio"], o["sink_num"], o["sink_den"], o["out_channels"])
    assert p.state_bytes == o["state_bytes"]
    assert p.latency == o["latency_sink"] * den // num
    assert p.macs_per_sample > 0
    assert "ops:" in p.describe()


def test_macs_match_survey():
    # cfg2 524,288 FLOP/frame; cfg4 49.8 kFLOP/sample; cfg5 79.9 kFLOP/sample
    assert Plan(configs.build(2), device=-1).macs_per_sample * 2 == 524288
    assert abs(Plan(configs.build(4), device=-1).macs_per_sample * 2 / 2048 - 49.8e3) < 0.1e3
    assert abs(Plan(configs.build(5), device=-1).macs_per_sample * 2 - 79.9e3) < 0.1e3


def test_causalize_arithmetic_matches_oracle():
    for S in range(1, 9):
        for R in range(0, 9):
            for Dc in range(0, 33):
                assert delay_for_stride(S, R, Dc) == po.delay_for_stride(S, R, Dc)
    assert branch_alignment([5, 2, 0]) == [0, 3, 5]
    for L, K, S, d in [(10, 3, 1, 1), (17, 4, 2, 3), (100, 9, 4, 1)]:
        assert conv_output_length(L, K, S, d) == po.oracle().oc_conv_output_length(L, K, S, d)
        if po.ref_available():
            assert conv_output_length(L, K, S, d) == po.ref().ref_conv_output_length(L, K, S, d)


def err_code(build):
    m = Model(4)
    build(m)
    with pytest.raises(StreamconvError) as e:
        Plan(m, device=-1)
    return e.value.code, str(e.value)


def test_typed_errors():
    assert err_code(lambda m: m.conv(3, 4, 3))[0] == "ChannelMismatch"
    assert err_code(lambda m: m.conv(4, 4, 3, padding=(1, 0)))[0] == "PaddingNotStreamable"
    assert err_code(lambda m: m.conv(4, 4, 9, stride=4, padding=(1, 1)))[0] == "PaddingNotStreamable"
    assert err_code(lambda m: m.conv_transpose(4, 4, 8, 4, padding=(1, 1)))[0] == "PaddingNotStreamable"

    def unclosed(m):
        m._node(3)
        m.conv(4, 4, 3)
    assert err_code(unclosed)[0] == "MalformedGraph"
    assert err_code(lambda m: m._node(4))[0] == "MalformedGraph"
    assert err_code(lambda m: m.gate())[0] == "UnsupportedFormat"
    assert err_code(lambda m: m._node(42))[0] == "SchemaError"
    assert err_code(lambda m: m.slice(2, 4))[0] == "ChannelMismatch"

    def rate_mismatch(m):
        m._node(3)
        m.conv(4, 4, 4, stride=2, padding=(2, 1))
        m._node(4)
    assert err_code(rate_mismatch)[0] == "RateMismatchAtSum"
    code, msg = err_code(lambda m: m.conv(3, 4, 3))
    assert msg.startswith("ChannelMismatch: ")  # streamconv::Error::what() format (error.hpp:59-60)


def test_bad_precision_and_state_on_host_plan():
    m = configs.build(1)
    nodes, n, w = m.pack()
    h = C.c_void_p()
    st = lib().sc_plan_create(nodes, n, w.ctypes.data_as(C.POINTER(C.c_float)), w.size, 64, 7, -1,
                              C.byref(h))
    assert st == 1  # InvalidArgument
    p = Plan(m, device=-1)
    from paper_2204_07064_b200.runtime import StreamState
    with pytest.raises(StreamconvError) as e:
        StreamState(p, 1, 2048)
    assert e.value.code == "InvalidArgument"


def test_weights_out_of_range():
    m = Model(2)
    m.conv(2, 2, 3)
    nodes, n, w = m.pack()
    h = C.c_void_p()
    st = lib().sc_plan_create(nodes, n, w.ctypes.data_as(C.POINTER(C.c_float)), w.size - 1, 2, 0, -1,
                              C.byref(h))
    assert st == 1 and b"weights" in lib().sc_last_error()


def test_pqmf_filters_design():
    from paper_2204_07064_b200.graph import pqmf_filters, pqmf_prototype
    ana, syn = pqmf_filters(16, 256)
    h = pqmf_prototype(16, 256)
    assert ana.shape == (16 * 256 + 16,) and syn.shape == (16 * 256 + 1,)
    assert abs(h.sum() - 1.0) < 1e-2              # unit DC gain lowpass
    assert np.allclose(h, h[::-1], atol=1e-12)    # linear phase
    # analysis filters are the time-reversed cosine-modulated prototype
    n = np.arange(256)
    k = 3
    hk = 2 * h * np.cos((2 * k + 1) * np.pi / 32 * (n - 127.5) + (-1) ** k * np.pi / 4)
    np.testing.assert_allclose(ana[k * 256:(k + 1) * 256], hk[::-1].astype(np.float32), atol=1e-7)


def test_pqmf_filters_match_independent_design():
    """The product's filter design (csrc/pqmf.cpp: Bessel series + golden-section search) is
    pinned to an independent numpy/scipy restatement of the published Kaiser-window PQMF
    design (oracle/pqmf_design.py: numpy.kaiser / numpy.sinc / numpy.correlate + bounded
    Brent) — the reference itself has no PQMF."""
    from oracle import pqmf_design as pd
    from paper_2204_07064_b200.graph import pqmf_filters, pqmf_prototype
    for M, N in ((16, 256), (4, 64), (8, 128)):
        p, wc = pd.design(M, N)
        np.testing.assert_allclose(pqmf_prototype(M, N), p, rtol=0, atol=1e-8)
        ana, syn = pqmf_filters(M, N)
        a2, s2 = pd.filters(M, N)
        np.testing.assert_allclose(ana, a2, rtol=0, atol=1e-7)
        np.testing.assert_allclose(syn / M, s2 / M, rtol=0, atol=1e-7)
        # the published design criterion: 2M-lag autocorrelation of the prototype vanishes
        assert pd.objective(M, N, wc, pd.kaiser_beta(100.0)) < 1e-4


def test_cpp_cached_module_api_host():
    """include/streamconv_b200.hpp (C++ cached-module API) builds plans host-only."""
    import subprocess
    from paper_2204_07064_b200 import build as B
    exe = B.build_cpp_tests()
    r = subprocess.run([str(exe), "host"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "OK host" in r.stdout, r.stdout + r.stderr


def test_densify_plan_time(monkeypatch):
    """Narrow stride-1 convs are lowered to super-row GEMMs at plan time (graph.cpp densify): two
    output frames per row, four for N <= 32 (the gated head); the algorithmic MAC count
    (SPEC's literal count, kernels.cpp:96-99 per output) does not change."""
    from paper_2204_07064_b200 import configs
    from paper_2204_07064_b200.runtime import Plan
    for cfg in (4, 5):
        p = Plan(configs.build(cfg), device=-1)
        ops = [l for l in p.describe().split("\n") if " gate" in l]
        assert len(ops) == 1 and " x4 " in ops[0] and "nout=128" in ops[0] and "taps=12" in ops[0], ops
        macs = p.macs_per_sample
        monkeypatch.setenv("SC_DENSIFY4", "0")
        p2 = Plan(configs.build(cfg), device=-1)
        ops2 = [l for l in p2.describe().split("\n") if " gate" in l]
        assert " x2 " in ops2[0] and "nout=64" in ops2[0], ops2
        assert p2.macs_per_sample == macs
        monkeypatch.setenv("SC_DENSIFY", "0")
        p3 = Plan(configs.build(cfg), device=-1)
        assert " x2 " not in p3.describe() and " x4 " not in p3.describe()
        assert p3.macs_per_sample == macs
        monkeypatch.delenv("SC_DENSIFY")
        monkeypatch.delenv("SC_DENSIFY4")

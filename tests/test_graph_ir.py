"""CPU: SPEC graph_ir / causalize / model_io on general DAGs.

The product's analyses (sc_graph_validate / compression_ratio / receptive_field / causalize /
latency, sc_plan_create_graph's host-only lowering, sc_model_load / save) are checked against
the SPEC examples, against the oracle's independent DAG restatement (oracle/oracle.cpp
`oc_dag_*`), and against impulse probing; the SPEC properties (equivalence after shift,
idempotence, stream == offline) run on the oracle over random DAGs."""
import json

import numpy as np
import pytest

from dag_models import random_graph
from oracle import pyoracle as po
from paper_2204_07064_b200 import StreamconvError, _abi, configs
from paper_2204_07064_b200.graph import Graph, SynthConfig, make_synthetic_rave, model_to_graph
from paper_2204_07064_b200.runtime import Plan

N_RANDOM = 200


def chain(strides=(), ups=(), C=1):
    g = Graph(C)
    x = g.source
    for s in strides:
        x = g.conv(x, C, C, 2 * s, stride=s, padding=(s, s - 1))
    for u in ups:
        x = g.zero_upsample(x, u)
        x = g.conv(x, C, C, 2 * u, padding=(u, u - 1))
    g.sink(x)
    return g


def code_of(fn):
    with pytest.raises(StreamconvError) as e:
        fn()
    return e.value.code, str(e.value)


# ------------------------------------------------------------------ SPEC examples
def test_validate_examples():
    # single chain Source -> Conv(S=2) -> Sink -> Sink ratio 1/2
    g = Graph(1)
    g.sink(g.conv(g.source, 1, 1, 2, stride=2, padding=(1, 0)))
    v = g.validate()
    assert v["rates"][-1] == (1, 2) and v["out_channels"] == 1
    # Source -> Fanout -> {Conv(S=2), Conv(S=4)} -> Sum -> RateMismatchAtSum
    g = Graph(1)
    a = g.conv(g.source, 1, 1, 2, stride=2, padding=(1, 0))
    b = g.conv(g.source, 1, 1, 4, stride=4, padding=(2, 1))
    g.sink(g.sum(a, b))
    code, msg = code_of(g.validate)
    assert code == "RateMismatchAtSum" and "node" in msg
    # encoder (4,4,2) + decoder (2,4,4) -> Sink ratio 1/1
    assert chain((4, 4, 2), (2, 4, 4)).validate()["rates"][-1] == (1, 1)


def test_compression_ratio_examples():
    assert chain((4, 4, 2)).compression_ratio() == 32
    assert chain(()).compression_ratio() == 1
    assert chain((2, 2), (2, 2)).compression_ratio() == 4


def test_receptive_field_examples():
    for pad, want in (((2, 0), (2, 0)), ((1, 1), (1, 1))):
        g = Graph(1)
        g.sink(g.conv(g.source, 1, 1, 3, padding=pad))
        assert g.receptive_field() == want
    g = Graph(1)  # two stacked centered K=3 -> (2, 2)
    g.sink(g.conv(g.conv(g.source, 1, 1, 3, padding=(1, 1)), 1, 1, 3, padding=(1, 1)))
    assert g.receptive_field() == (2, 2)


def test_causalize_and_latency_examples():
    # already-causal chain -> identical graph, latency 0
    g = Graph(1)
    g.sink(g.conv(g.conv(g.source, 1, 1, 3, padding=(2, 0)), 1, 1, 3, padding=(2, 0)))
    gc, lat = g.causalize()
    assert lat == 0 and len(gc.nodes) == len(g.nodes) and g.latency() == 0
    # centered K=3 -> pad (2, 0), latency 1; latency_of(causalized) = 1
    g = Graph(1)
    g.sink(g.conv(g.source, 1, 1, 3, padding=(1, 1)))
    gc, lat = g.causalize()
    conv = [n for n in gc.nodes if n["kind"] == _abi.G_CONV][0]
    assert lat == 1 and (conv["pad_left"], conv["pad_right"]) == (2, 0)
    assert gc.receptive_field()[1] == 0 and gc.latency() == 1
    # latency_of a non-causal graph -> NotCausal
    assert code_of(g.latency)[0] == "NotCausal"


def test_rave_post_vs_pre_training_causal_latency():
    """post-training causalized latency >> pre-training causal (stride residue)."""
    post = make_synthetic_rave(SynthConfig(padding="centered")).causalize()[1]
    pre = make_synthetic_rave(SynthConfig(padding="causal")).latency()
    assert post > 10 * max(pre, 1) and pre < 32


# ------------------------------------------------------------------ validate errors
def test_validate_error_categories():
    g = Graph(2)
    a = g.conv(g.source, 2, 2, 1, padding=(0, 0))
    b = g.conv(a, 2, 2, 1, padding=(0, 0))
    g.sink(b)
    g.edges.append((b, a, 0))  # second edge into a's port 0
    assert code_of(g.validate)[0] == "MalformedGraph"
    # a cycle: Sum(source, b) -> a -> b -> Sum
    g = Graph(2)
    s = g.add(_abi.G_SUM, [g.source], arity=2)
    a = g.conv(s, 2, 2, 1, padding=(0, 0))
    g.sink(a)
    g.edges.append((a, s, 1))
    code, msg = code_of(g.validate)
    assert code == "CycleDetected" and "node" in msg
    # channel mismatch, named node
    g = Graph(2)
    g.sink(g.conv(g.source, 3, 2, 1, padding=(0, 0)))
    code, msg = code_of(g.validate)
    assert code == "ChannelMismatch" and "node 1" in msg
    # a node that never reaches the Sink
    g = Graph(2)
    g.conv(g.source, 2, 2, 1, padding=(0, 0))
    g.sink(g.source)
    assert code_of(g.validate)[0] in ("DanglingNode", "MalformedGraph")
    g = Graph(2)  # unknown kind
    g.sink(g.add(42, [g.source]))
    assert code_of(g.validate)[0] == "SchemaError"
    g = Graph(2)  # no sink
    g.conv(g.source, 2, 2, 1, padding=(0, 0))
    assert code_of(g.validate)[0] in ("MalformedGraph", "DanglingNode")


def test_validate_is_total_on_mutations():
    """every malformed graph yields a typed error, never a crash."""
    rng = np.random.default_rng(3)
    for seed in range(60):
        g = random_graph(seed).finalized()
        for _ in range(3):
            h = Graph.from_arrays(*g.pack(), g.in_channels)
            m = rng.integers(0, 4)
            if m == 0 and h.edges:
                h.edges.pop(int(rng.integers(0, len(h.edges))))
            elif m == 1 and h.edges:
                a, b, p = h.edges[int(rng.integers(0, len(h.edges)))]
                h.edges.append((b, a, p))
            elif m == 2:
                i = int(rng.integers(0, len(h.nodes)))
                h.nodes[i]["in_channels"] += 1
            else:
                h.edges.append((int(rng.integers(0, len(h.nodes))), int(rng.integers(0, len(h.nodes))),
                                int(rng.integers(0, 3))))
            try:
                h.validate()
            except StreamconvError as e:
                assert e.code in _abi.ERR_NAMES


# ------------------------------------------------------------------ product vs oracle
def test_flat_and_dag_lowering_identical_for_configs():
    for cfg in (1, 2, 3, 4, 5):
        m = configs.build(cfg, seed=0)
        p1, p2 = Plan(m, device=-1), Plan(model_to_graph(m), device=-1)
        d1 = _abi.lib().sc_plan_describe(p1._h).decode()
        d2 = _abi.lib().sc_plan_describe(p2._h).decode()
        assert d1 == d2, cfg


@pytest.mark.parametrize("chunk", range(4))
def test_random_dags_product_analyses_match_oracle(chunk):
    for seed in range(chunk * N_RANDOM // 4, (chunk + 1) * N_RANDOM // 4):
        g = random_graph(seed)
        info = po.graph_info(g)
        p = Plan(g, device=-1)
        assert p.ratio == info["ratio"] == g.compression_ratio(), seed
        num, den, oc = p.sink
        assert (num, den, oc) == (info["sink_num"], info["sink_den"], info["out_channels"]), seed
        assert p.latency == info["latency_in"] == g.causalize()[1], seed
        assert p.state_bytes == info["state_bytes"], seed


def _impulse_support(g, T, t0):
    x = np.zeros((1, g.in_channels, T), np.float32)
    x[0, :, t0] = 1.0
    y = po.run(g, x, mode="offline_original")[0]
    nz = np.nonzero(np.abs(y).max(axis=0) > 0)[0]
    return nz.min(), nz.max()


def test_receptive_field_vs_impulse_probe():
    """exact agreement with impulse probing (linear graphs, random weights)."""
    checked = 0
    for seed in range(400):
        g = random_graph(seed, linear=True, max_den=1)  # stride-1 graphs: probing is exact
        past, fut = g.receptive_field()
        T = 4 * (past + fut) + 64
        t0 = T // 2
        lo, hi = _impulse_support(g, T, t0)
        if all(n["kind"] != _abi.G_DELAY for n in g.nodes):
            assert (hi - t0, t0 - lo) == (past, fut), seed
        else:  # a Delay shifts the support: future may be negative (clamped at 0)
            assert hi - t0 == past and max(0, t0 - lo) == fut, seed
        checked += 1
    assert checked >= 300


# ------------------------------------------------------------------ SPEC properties on the oracle
def _shift_check(g, T=None, seed=0):
    gc, lat_in = g.causalize()
    past, fut = g.receptive_field()
    r = g.compression_ratio()
    info = po.graph_info(g)
    num, den = info["sink_num"], info["sink_den"]
    lat = lat_in * num // den  # the shift in sink frames
    T = T or r * max(8, -(-4 * (past + fut + lat_in + 8) // r))
    x = np.random.default_rng(seed).standard_normal((1, g.in_channels, T)).astype(np.float32)
    yo = po.run(g, x, mode="offline_original")[0]
    yc = po.run(g, x, mode="offline")[0]
    m = -(-(past + fut + r) * num // den) + 1  # sink frames touched by the signal edges
    a, b = m + lat, yo.shape[-1] - lat - m
    if b <= a:
        return False
    ref = yo[:, a - lat:b - lat]
    err = np.abs(yc[:, a:b] - ref).max()
    assert err <= 1e-5 * max(1.0, float(np.abs(ref).max())), (err, lat)
    return True


@pytest.mark.parametrize("chunk", range(4))
def test_equivalence_after_shift_random_dags(chunk):
    """offline_run(causalize(g)) == shift(offline_run(g), latency) (interior)."""
    done = 0
    for seed in range(chunk * N_RANDOM // 4, (chunk + 1) * N_RANDOM // 4):
        done += _shift_check(random_graph(seed), seed=seed)
    assert done >= N_RANDOM // 8


def test_causalize_idempotent_random_dags():
    for seed in range(N_RANDOM):
        g = random_graph(seed)
        gc, lat = g.causalize()
        gcc, lat2 = gc.causalize()
        assert lat2 == lat and len(gcc.nodes) == len(gc.nodes), seed
        assert gc.receptive_field()[1] == 0 and gc.latency() == lat, seed


@pytest.mark.parametrize("pad", ["centered", "causal"])
def test_synthetic_rave(pad):
    g = make_synthetic_rave(SynthConfig(padding=pad))
    past, fut = g.receptive_field()
    assert (fut == 0) == (pad == "causal")
    h = make_synthetic_rave(SynthConfig(padding=pad))
    assert all(np.array_equal(a, b) for a, b in zip(g.chunks, h.chunks))  # determinism
    assert _shift_check(g)
    # streaming == offline causalized, any multiple-of-ratio partition
    r = g.compression_ratio()
    x = np.random.default_rng(1).standard_normal((2, 1, 24 * r)).astype(np.float32)
    y_off = po.run(g, x, mode="offline")
    for parts in ([24 * r], [r] * 24, [8 * r, 2 * r, 14 * r]):
        assert np.array_equal(po.run(g, x, parts, "stream"), y_off)


def test_stream_equals_offline_random_dags():
    for seed in range(0, N_RANDOM, 4):
        g = random_graph(seed)
        r = g.compression_ratio()
        x = np.random.default_rng(seed).standard_normal((1, g.in_channels, 12 * r)).astype(np.float32)
        y_off = po.run(g, x, mode="offline")
        assert np.array_equal(po.run(g, x, [r] * 12, "stream"), y_off), seed
        assert np.array_equal(po.run(g, x, [5 * r, 7 * r], "stream"), y_off), seed


def test_flat_model_and_dag_oracles_agree():
    """The oracle's flat (node list) and DAG restatements give bit-identical streams."""
    for cfg in (1, 2, 3):
        m = configs.build(cfg, seed=0)
        g = model_to_graph(m)
        r = po.graph_info(m)["ratio"]
        T = r * (8 if cfg != 3 else 2)
        x = configs.batch_input(cfg, range(1), m.in_channels, T, seed=0)
        assert np.array_equal(po.run(m, x, [T // 2, T // 2]), po.run(g, x, [T // 2, T // 2])), cfg


# ------------------------------------------------------------------ model_io
def test_model_io_round_trip(tmp_path):
    for seed in range(10):
        g = random_graph(seed).finalized()
        g.save(tmp_path / "model.json")
        assert (tmp_path / "model.bin").exists()
        h = Graph.load(tmp_path / "model.json")
        assert len(h.nodes) == len(g.nodes) and h.edges == g.edges
        for a, b in zip(g.nodes, h.nodes):
            fields = {_abi.G_CONV: ("in_channels", "out_channels", "taps", "stride", "dilation",
                                    "pad_left", "pad_right", "shift", "hint"),
                      _abi.G_ZERO_UPSAMPLE: ("factor",), _abi.G_ACTIVATION: ("act",),
                      _abi.G_DELAY: ("samples", "inserted"), _abi.G_SUM: ("arity",),
                      _abi.G_FANOUT: ("arity",), _abi.G_SLICE: ("slice_begin", "slice_count")}
            assert a["kind"] == b["kind"]
            for k in fields.get(a["kind"], ()):
                assert a[k] == b[k], (seed, k)
            if a["kind"] == _abi.G_ACTIVATION:
                assert np.float32(a["alpha"]) == np.float32(b["alpha"])
        x = np.random.default_rng(seed).standard_normal((1, g.in_channels, 8 * g.compression_ratio()))
        x = x.astype(np.float32)
        assert np.array_equal(po.run(g, x, mode="offline"), po.run(h, x, mode="offline"))
    m = json.loads((tmp_path / "model.json").read_text())
    assert m["format_version"] == 1 and m["nodes"][0]["kind"] == "Source"


def _write(tmp_path, manifest, blob=b""):
    (tmp_path / "m.json").write_text(json.dumps(manifest))
    (tmp_path / "m.bin").write_bytes(blob)
    return tmp_path / "m.json"


def test_model_io_errors(tmp_path):
    g = Graph(1)
    g.sink(g.conv(g.source, 1, 2, 3, padding=(1, 1)))
    g.save(tmp_path / "ok.json")
    man = json.loads((tmp_path / "ok.json").read_text())
    blob = (tmp_path / "ok.bin").read_bytes()
    assert len(blob) == (2 * 1 * 3 + 2) * 4
    # truncated blob -> CorruptBlob
    p = _write(tmp_path, man, blob[:-4])
    assert code_of(lambda: Graph.load(p))[0] == "CorruptBlob"
    p = _write(tmp_path, man, blob + b"\0\0\0\0")
    assert code_of(lambda: Graph.load(p))[0] == "CorruptBlob"
    # unknown node kind -> SchemaError naming the kind and its JSON path
    bad = json.loads(json.dumps(man))
    bad["nodes"][1]["kind"] = "Reverb"
    code, msg = code_of(lambda: Graph.load(_write(tmp_path, bad, blob)))
    assert code == "SchemaError" and "Reverb" in msg and "$.nodes[1].kind" in msg
    bad = json.loads(json.dumps(man))
    del bad["nodes"][1]["kernel"]
    code, msg = code_of(lambda: Graph.load(_write(tmp_path, bad, blob)))
    assert code == "SchemaError" and "$.nodes[1].kernel" in msg
    bad = json.loads(json.dumps(man))
    bad["format_version"] = 2
    assert code_of(lambda: Graph.load(_write(tmp_path, bad, blob)))[0] == "VersionMismatch"
    # a manifest whose graph fails validate -> the validate category
    bad = json.loads(json.dumps(man))
    bad["nodes"][1]["in_channels"] = 3
    bad["nodes"][1]["weights"]["length"] = (2 * 3 * 3 + 2) * 4
    assert code_of(lambda: Graph.load(_write(tmp_path, bad, b"\0" * ((2 * 3 * 3 + 2) * 4))))[0] == \
        "ChannelMismatch"
    (tmp_path / "broken.json").write_text("{\"format_version\": 1, ")
    (tmp_path / "broken.bin").write_bytes(b"")
    assert code_of(lambda: Graph.load(tmp_path / "broken.json"))[0] == "SchemaError"

"""Out-of-bounds write detection without compute-sanitizer (closed on the GPU pool): states
created with SC_REDZONE=1 carry guard bytes after every stream's strip and around every buffer
(sc_state_redzone_check), and the caller's output tensors get guard elements here.  Runs the
machinery the kernels share — strip wrap-around (carry, SC_STRIP_K=3), subset and full reset,
phase state (cfg5 B = 512), window / X2 / chained tensor-core tiles, PQMF, bf16 storage —
and requires every guard to be intact."""
import numpy as np
import pytest

from paper_2204_07064_b200 import configs
from paper_2204_07064_b200.runtime import Plan, StreamState

torch = pytest.importorskip("torch")

CASES = [  # cfg, precision, streams, parts, reset-after-call (None: full reset at the end)
    (2, "fp32", 3, [512, 256, 512, 768, 1024], 1),
    (3, "fp32", 2, [1024, 1024, 2048, 1024], 1),
    (4, "fp32", 5, [1] * 6, 2),
    (5, "fp32", 2, [2048, 2048, 2048, 2048], 1),
    (5, "fp32", 3, [512] * 8, 3),          # phase state; subset reset at a period boundary
    (2, "bf16", 2, [512, 512, 1024], 1),
    (5, "bf16", 2, [2048, 2048], None),
]


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,prec,S,parts,rst", CASES,
                         ids=[f"cfg{c[0]}-{c[1]}-{len(c[3])}x{c[3][0]}" for c in CASES])
def test_no_out_of_bounds_writes(cfg, prec, S, parts, rst, monkeypatch):
    monkeypatch.setenv("SC_REDZONE", "1")
    monkeypatch.setenv("SC_STRIP_K", "3")
    m = configs.build(cfg, seed=cfg)
    x = configs.batch_input(cfg, range(S), m.in_channels, sum(parts), seed=cfg)
    plan = Plan(m, precision=prec)
    num, den, cout = plan.sink
    st = StreamState(plan, S, max(parts))
    assert st.redzone_violations() == 0
    xd = torch.from_numpy(x).cuda()
    G = 4096  # guard elements after the caller's output
    t0 = 0
    for j, p in enumerate(parts):
        n_out = S * cout * (p * num // den)
        buf = torch.full((n_out + G,), 12345.0, device="cuda")
        y = buf[:n_out].view(S, cout, p * num // den)
        st.set_graphs(j % 2 == 0)
        st.process_buffer(xd[:, :, t0:t0 + p].contiguous(), y, p)
        torch.cuda.synchronize()
        assert torch.isfinite(y).all()
        assert bool((buf[n_out:] == 12345.0).all()), f"call {j}: write past the output tensor"
        t0 += p
        if rst is not None and j == rst:
            st.reset([S - 1])
    assert st.redzone_violations() == 0
    st.reset()
    assert st.redzone_violations() == 0


@pytest.mark.gpu
def test_redzone_detects_a_stray_write(monkeypatch):
    """The checker itself: bytes written into the state's tail guard are counted."""
    import ctypes as C
    from paper_2204_07064_b200._abi import lib
    rt = pytest.importorskip("cuda.bindings.runtime")
    monkeypatch.setenv("SC_REDZONE", "1")
    st = StreamState(Plan(configs.build(2, seed=1)), 2, 512)
    assert st.redzone_violations() == 0
    f = lib().sc_debug_state_mem
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]
    ptr, nbytes = C.c_void_p(), C.c_int64()
    assert f(st._h, C.byref(ptr), C.byref(nbytes)) == 0
    torch.cuda.synchronize()
    (err,) = rt.cudaMemset(ptr.value + nbytes.value - 100, 0, 8)
    assert int(err) == 0
    torch.cuda.synchronize()
    assert st.redzone_violations() == 8

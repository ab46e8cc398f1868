"""Random SPEC graph_ir DAGs for the graph_ir / causalize property tests (SPEC.md:228-233:
"200 random valid graphs (depth <= 6, strides in {1,2,4}, K <= 8, with/without residual
branches and upsampling)").  Every generated graph is valid, streamable (conv pads total
(K-1)d, strided pads >= span - S) and lowerable by the product (ZeroUpsample feeds a stride-1,
dilation-1 conv with pads totalling K-1)."""
from __future__ import annotations

import numpy as np

from paper_2204_07064_b200._abi import ACT_IDENTITY, ACT_LEAKY_RELU, ACT_TANH
from paper_2204_07064_b200.graph import Graph


def _split(rng, tot, centered_p=0.5):
    if rng.random() < centered_p:
        return ((tot + 1) // 2, tot // 2)
    left = int(rng.integers(0, tot + 1))
    return (left, tot - left)


def random_graph(seed: int, depth: int = 6, channels=(2, 3, 4), linear: bool = False,
                 max_den: int = 8, init: str = "kaiming") -> Graph:
    """A random DAG.  `linear`: identity activations only (impulse-probing tests)."""
    rng = np.random.default_rng(seed)
    C = int(rng.choice(channels))
    g = Graph(C, seed=seed)
    x = g.source
    den, num = 1, 1  # rate of x relative to the source

    def conv_s1(x, cin, cout, kmax=8):
        k = int(rng.integers(1, kmax + 1))
        d = int(rng.integers(1, 4)) if k > 1 and rng.random() < 0.4 else 1
        return g.conv(x, cin, cout, k, dilation=d, padding=_split(rng, (k - 1) * d), init=init)

    def act(x):
        if linear:
            return x
        kind = int(rng.choice([ACT_LEAKY_RELU, ACT_TANH]))
        return g.act(x, kind, 0.2)

    for _ in range(int(rng.integers(1, depth + 1))):
        op = rng.choice(["conv", "strided", "up", "res", "branch3", "delay", "act", "downup"])
        C2 = int(rng.choice(channels))
        if op == "conv":
            x = conv_s1(x, C, C2)
            C = C2
        elif op == "strided" and den * 4 <= max_den:
            S = int(rng.choice([2, 4]))
            k = int(rng.integers(S, min(2 * S + 1, 8) + 1))
            P = int(rng.integers(k - S, k))  # span - S <= P <= span - 1
            x = g.conv(x, C, C2, k, stride=S, padding=_split(rng, P), init=init)
            den *= S
            C = C2
        elif op == "up" and den > 1:
            f = 2 if den % 4 else int(rng.choice([2, 4]))
            x = g.zero_upsample(x, f)
            k = 2 * f
            x = g.conv(x, C, C2, k, padding=_split(rng, k - 1), init=init)
            den //= f
            C = C2
        elif op == "res":
            h = act(x)
            h = conv_s1(h, C, C, kmax=5)
            if rng.random() < 0.5:
                h = conv_s1(act(h), C, C, kmax=1)
            skip = g.delay(x, int(rng.integers(1, 4))) if rng.random() < 0.3 else x
            x = g.sum(h, skip) if rng.random() < 0.7 else g.sum(skip, h)
        elif op == "branch3":
            a = conv_s1(act(x), C, C, kmax=4)
            b = conv_s1(x, C, C, kmax=6)
            x = g.sum(a, b, x)
        elif op == "downup" and den * 2 <= max_den:
            # a residual branch that changes rate inside (stride 2 down, x2 up)
            h = g.conv(act(x), C, C, 3, stride=2, padding=_split(rng, int(rng.integers(1, 3))), init=init)
            h = g.zero_upsample(h, 2)
            h = g.conv(h, C, C, 4, padding=_split(rng, 3), init=init)
            x = g.sum(x, h)
        elif op == "delay":
            x = g.delay(x, int(rng.integers(0, 5)))
        elif op == "act":
            x = act(x)
    if rng.random() < 0.3:
        x = g.delay(x, int(rng.integers(1, 3)))
    g.sink(x)
    return g

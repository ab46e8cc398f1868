"""Small graphs whose reference-conv streaming outputs are pinned in ref_stream.npz."""
from paper_2204_07064_b200.graph import Model


def small_models():
    m1 = Model(4, 1)
    m1.conv(4, 4, 3, padding=(1, 1))
    m2 = Model(3, 2)
    with m2.residual():
        m2.leaky_relu(0.2)
        m2.conv(3, 3, 3, dilation=2, padding=(2, 2))
        m2.leaky_relu(0.2)
        m2.conv(3, 3, 1, padding=(0, 0))
    m3 = Model(2, 3)
    m3.conv(2, 4, 9, stride=4, padding=(4, 4)).leaky_relu(0.2).conv(4, 6, 5, stride=2, padding=(2, 2))
    m3.leaky_relu(0.2).conv_transpose(6, 4, 4, 2, padding=(2, 1)).leaky_relu(0.2)
    m3.conv_transpose(4, 2, 8, 4, padding=(4, 3))
    return dict(centered=m1, residual=m2, encdec=m3)

"""streamconv-b200: B200-native multi-stream cached-padding streaming inference
(the hot path of arXiv 2204.07064, SPEC stream_runtime) behind a C-ABI."""
from ._abi import StreamconvError, lib  # noqa: F401
from .graph import Model  # noqa: F401
from .runtime import Plan, StreamState, conv1d  # noqa: F401

__all__ = ["Model", "Plan", "StreamState", "StreamconvError", "conv1d", "lib"]

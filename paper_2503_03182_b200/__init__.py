"""paper_2503_03182_b200 — B200-native TPipe hot path (T-Pipe + T-Recomp +
T-Offload) behind the C-ABI of include/tpipe.h. See DESIGN.md."""

from ._lib import LIB_PATH, TPipeError, lib  # noqa: F401

"""B200-native (sm_100a) segregated 2x transpose convolution.

Drop-in for the reference ``segconv`` operator path (arXiv 2209.03704):
``segregate`` + ``transpose_conv_fused`` with ``transpose_conv_naive`` selectable
as the conventional baseline.  See DESIGN.md.
"""
from .segconv import *  # noqa: F401,F403
from .segconv import __all__ as _seg_all

__all__ = list(_seg_all)

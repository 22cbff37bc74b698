"""paper_2008_10275_b200 -- B200-native truncated low-rank ChebyshevT (arxiv 2008.10275).

The product is the C-ABI library ``liblrcheb.so`` (include/lrcheb.h; CUDA kernels for sm_100a in
``csrc/``); ``lrcheb`` is its thin ctypes binding.  Importing the binding raises if the library
is missing -- there is no CPU fallback.
"""
from . import lrcheb  # noqa: F401
from .lrcheb import Context, LrcError, version  # noqa: F401

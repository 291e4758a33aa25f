"""B200-native FDA Burton-Miller apply (arXiv 1311.5202): libfda.so + ctypes binding.

The product is the C-ABI library ``libfda.so`` (include/fda.h) built from
``csrc/`` for sm_100a; ``fda`` is its thin Python binding.  See DESIGN.md.
"""
from . import fda  # noqa: F401  (raises ImportError if libfda.so is not built)
from .fda import Plan  # noqa: F401

"""B200-native FDA Burton-Miller apply (arXiv 1311.5202): libfda.so + ctypes binding.

The product is the C-ABI library ``libfda.so`` (include/fda.h) built from
``csrc/`` for sm_100a (``python -m paper_1311_5202_b200.build``); its thin Python
binding is ``paper_1311_5202_b200.fda`` (importing it raises ImportError if the
library is not built -- there is no fallback).  See DESIGN.md.
"""

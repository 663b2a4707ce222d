"""fdsdf -- B200-native finite-difference curvature regularisation for neural SDFs
(arXiv 2511.08980).  The compute path is libfdsdf.so (hand-written sm_100a CUDA, C ABI in
include/fdsdf.h); this package is its thin Python binding plus data-parallel host glue."""
from .fdsdf import *  # noqa: F401,F403
from .fdsdf import FDSDF, FdsdfError, lib, version  # noqa: F401

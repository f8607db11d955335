"""vtc-b200: B200-native executor for VTC-planned graphs (arXiv 2604.09558).

Data-movement operators become VirtualTensor div/mod maps evaluated inside
sm_100a consumer kernels; see DESIGN.md.  The compute path is libvtc.so
(C++ host + CUDA); this package is a thin ctypes mirror of its C ABI.
"""
from .api import (  # noqa: F401
    CompGraph, Comm, Plan, VtcError, ERRORS, execute, parse_graph, f32_to_bf16, bf16_to_f32,
    MATERIALIZE, SELECTED, MAX_ELIMINATION, INPLACE_UPDATES, GREEDY, FLAG_FAST_FP, FLAG_NO_GEMV, FLAG_NO_FUSE, FLAG_GEMV_LDG, FLAG_NO_TC, FLAG_DYNAMIC_POS,
    NP_DTYPES,
)
from .api import ERRORS as _ERRORS

globals().update({cls.__name__: cls for cls in _ERRORS.values()})  # UnsupportedError, SchemaError, ...

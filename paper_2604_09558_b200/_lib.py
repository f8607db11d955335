"""ctypes binding of libvtc.so (include/vtc.h).

The product path is this native library.  If it is missing the import fails
loudly -- there is no Python or CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libvtc.so"

# Every symbol declared in include/vtc.h: name -> (restype, argtypes)
_VP = C.c_void_p
SIGNATURES = {
    "vtc_last_error": (C.c_char_p, []),
    "vtc_version": (C.c_char_p, []),
    "vtc_graph_parse": (C.c_int, [C.c_char_p, C.POINTER(_VP)]),
    "vtc_graph_free": (None, [_VP]),
    "vtc_graph_serialize": (C.c_int, [_VP, C.POINTER(C.c_char_p)]),
    "vtc_graph_vtog": (C.c_int, [_VP, C.POINTER(C.c_char_p)]),
    "vtc_graph_estimate": (C.c_int, [_VP, C.POINTER(C.c_int32), C.c_int32, C.c_char_p, C.POINTER(C.c_char_p)]),
    "vtc_graph_enumerate": (C.c_int, [_VP, C.c_int64, C.POINTER(C.c_char_p)]),
    "vtc_graph_greedy": (C.c_int, [_VP, C.c_char_p, C.POINTER(C.c_char_p)]),
    "vtc_plan_create": (C.c_int, [_VP, C.c_int, C.POINTER(C.c_int32), C.c_int32, C.c_uint32, C.POINTER(_VP)]),
    "vtc_plan_free": (None, [_VP]),
    "vtc_plan_info": (C.c_int, [_VP, C.c_int, C.POINTER(C.c_char_p)]),
    "vtc_plan_bind_root": (C.c_int, [_VP, C.c_char_p, _VP]),
    "vtc_plan_root_ptr": (C.c_int, [_VP, C.c_char_p, C.POINTER(_VP)]),
    "vtc_plan_upload": (C.c_int, [_VP, C.c_char_p, _VP, C.c_int64, _VP]),
    "vtc_plan_download": (C.c_int, [_VP, C.c_char_p, _VP, C.c_int64, _VP]),
    "vtc_run": (C.c_int, [_VP, C.c_int32, C.POINTER(C.c_char_p), C.POINTER(_VP), C.POINTER(C.c_int64),
                          C.c_int32, C.POINTER(C.c_char_p), C.POINTER(_VP), C.POINTER(C.c_int64), _VP]),
    "vtc_plan_prepare": (C.c_int, [_VP]),
    "vtc_plan_set_position": (C.c_int, [_VP, C.c_int64, _VP]),
    "vtc_execute": (C.c_int, [_VP, _VP]),
    "vtc_execute_graph": (C.c_int, [_VP, _VP]),
    "vtc_plan_num_launches": (C.c_int, [_VP]),
    "vtc_execute_timed": (C.c_int, [_VP, _VP, C.POINTER(C.c_float), C.c_int32]),
    "vtc_plan_trace": (C.c_int, [_VP, C.POINTER(C.c_uint64), C.c_int32]),
    "vtc_map_eval": (C.c_int, [_VP, C.c_char_p, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.c_int64]),
    "vtc_plan_map_json": (C.c_int, [_VP, C.c_char_p, C.POINTER(C.c_char_p)]),
    "vtc_plan_map_analyze": (C.c_int, [_VP, C.c_char_p, C.c_int64, C.c_int64, C.POINTER(C.c_char_p)]),
    "vtc_comm_unique_id": (C.c_int, [_VP, C.c_int32]),
    "vtc_comm_init": (C.c_int, [_VP, C.c_int32, C.c_int32, C.c_int32, C.POINTER(_VP)]),
    "vtc_comm_init_host": (C.c_int, [_VP, _VP, C.c_int32, C.c_int32, C.POINTER(_VP)]),
    "vtc_comm_free": (None, [_VP]),
    "vtc_plan_set_comm": (C.c_int, [_VP, _VP]),
    "vtc_launch_gather_copy": (C.c_int, [_VP, _VP, C.c_int32, _VP]),
}

_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the executor has no CPU fallback)"
        )
    lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib

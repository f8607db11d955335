"""ctypes wrapper of oracle/_ref/libvtelim_ref.so: the UNMODIFIED reference
library (built by oracle/Makefile from /root/reference sources) plus the
test-only C harness oracle/ref_capi.cpp.

TEST INFRASTRUCTURE ONLY (checker and timed CPU baseline).  Never imported by
the product package.
"""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path
from typing import Dict, Iterable, Optional

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libvtelim_ref.so"
DT_CODE = {"f64": 0, "f32": 1, "i64": 2}
NP = {"f64": np.float64, "f32": np.float32, "i64": np.int64}

_lib = None


def available() -> bool:
    return LIB.exists()


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(str(LIB))
        vp = C.c_void_p
        sig = {
            "vref_last_error": (C.c_char_p, []),
            "vref_graph_parse": (vp, [C.c_char_p]),
            "vref_graph_free": (None, [vp]),
            "vref_graph_serialize": (C.c_char_p, [vp]),
            "vref_vtog_json": (C.c_char_p, [vp]),
            "vref_ptg_all_physical": (vp, [vp]),
            "vref_ptg_validate": (vp, [vp, C.POINTER(C.c_int), C.c_int]),
            "vref_ptg_free": (None, [vp]),
            "vref_ptg_json": (C.c_char_p, [vp]),
            "vref_estimate_json": (C.c_char_p, [vp, vp]),
            "vref_estimate_params_json": (C.c_char_p, [vp, vp, C.c_char_p]),
            "vref_saving": (C.c_int, [vp, vp, C.c_char_p, C.POINTER(C.c_double)]),
            "vref_enumerate_json": (C.c_char_p, [vp, C.c_int64]),
            "vref_gather_map_json": (C.c_char_p, [vp, C.c_char_p, C.c_char_p]),
            "vref_map_eval_all": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.c_int64]),
            "vref_map_compose": (C.c_char_p, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int]),
            "vref_map_analyze": (C.c_char_p, [C.c_char_p, C.c_int64, C.c_int64]),
            "vref_inputs_random": (vp, [vp, C.c_uint64]),
            "vref_tensors_new": (vp, []),
            "vref_tensors_free": (None, [vp]),
            "vref_tensor_set": (C.c_int, [vp, C.c_char_p, C.c_int, C.POINTER(C.c_int64), C.c_int, vp]),
            "vref_tensor_bytes": (C.c_int64, [vp, C.c_char_p]),
            "vref_tensor_get": (C.c_int, [vp, C.c_char_p, vp, C.c_int64]),
            "vref_tensor_digest": (C.c_uint64, [vp, C.c_char_p]),
            "vref_execute": (vp, [vp, vp, vp, C.c_int, C.POINTER(C.c_double)]),
            "vref_last_skipped": (C.c_char_p, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class RefError(RuntimeError):
    pass


def _err():
    raise RefError(lib().vref_last_error().decode())


class RefGraph:
    def __init__(self, doc):
        self.text = doc if isinstance(doc, str) else json.dumps(doc)
        self.doc = json.loads(self.text)
        self.h = lib().vref_graph_parse(self.text.encode())
        if not self.h:
            _err()
        ser = json.loads(lib().vref_graph_serialize(self.h).decode())
        self.specs = {t["id"]: t for t in ser["tensors"]}

    def __del__(self):
        if getattr(self, "h", None):
            lib().vref_graph_free(self.h)

    def vtog(self) -> dict:
        s = lib().vref_vtog_json(self.h)
        if s is None:
            _err()
        return json.loads(s.decode())

    def plan(self, selected: Optional[Iterable[int]] = None) -> "RefPlan":
        if selected is None:
            h = lib().vref_ptg_all_physical(self.h)
        else:
            sel = list(selected)
            arr = (C.c_int * max(1, len(sel)))(*sel)
            h = lib().vref_ptg_validate(self.h, arr, len(sel))
        if not h:
            _err()
        return RefPlan(self, h)

    def enumerate_ptgs(self, limit: int = -1) -> list:
        s = lib().vref_enumerate_json(self.h, int(limit))
        if s is None:
            _err()
        return json.loads(s.decode())

    def gather_map(self, node: str, output: str) -> dict:
        s = lib().vref_gather_map_json(self.h, node.encode(), output.encode())
        if s is None:
            _err()
        return json.loads(s.decode())

    def inputs_random(self, seed: int = 1) -> Dict[str, np.ndarray]:
        t = lib().vref_inputs_random(self.h, seed)
        if not t:
            _err()
        try:
            return {tid: _get(t, tid, self.specs[tid]) for tid, s in self.specs.items() if s["kind"] == "input"}
        finally:
            lib().vref_tensors_free(t)


class RefPlan:
    def __init__(self, g: RefGraph, h):
        self.g = g
        self.h = h
        self.info = json.loads(lib().vref_ptg_json(h).decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().vref_ptg_free(self.h)

    def estimate(self) -> dict:
        s = lib().vref_estimate_json(self.g.h, self.h)
        if s is None:
            _err()
        return json.loads(s.decode())

    def estimate_params(self, params: dict) -> dict:
        s = lib().vref_estimate_params_json(self.g.h, self.h, json.dumps(params).encode())
        if s is None:
            _err()
        return json.loads(s.decode())

    def saving(self, params: dict) -> float:
        out = C.c_double()
        if lib().vref_saving(self.g.h, self.h, json.dumps(params).encode(), C.byref(out)):
            _err()
        return out.value

    def execute(self, inputs: Dict[str, np.ndarray], with_roots: bool = False):
        """Returns (outputs, wall_ns, skipped_ops)."""
        t = lib().vref_tensors_new()
        try:
            for tid, a in inputs.items():
                spec = self.g.specs[tid]
                a = np.ascontiguousarray(a, dtype=NP[spec["dtype"]])
                shp = (C.c_int64 * max(1, a.ndim))(*a.shape)
                if lib().vref_tensor_set(t, tid.encode(), DT_CODE[spec["dtype"]], shp, a.ndim,
                                         a.ctypes.data_as(C.c_void_p)):
                    _err()
            ns = C.c_double(0)
            o = lib().vref_execute(self.g.h, self.h, t, 1 if with_roots else 0, C.byref(ns))
            if not o:
                _err()
            skipped = [s for s in lib().vref_last_skipped().decode().split("\n") if s]
            try:
                out = {}
                for tid, spec in self.g.specs.items():
                    if spec["kind"] == "output":
                        out[tid] = _get(o, tid, spec)
                if with_roots:
                    for tid in self.info["roots"]:
                        out["root:" + tid] = _get(o, "root:" + tid, self.g.specs[tid])
                return out, ns.value, skipped
            finally:
                lib().vref_tensors_free(o)
        finally:
            lib().vref_tensors_free(t)


def _get(t, tid: str, spec: dict) -> np.ndarray:
    out = np.empty(spec["shape"], dtype=NP[spec["dtype"]])
    if lib().vref_tensor_get(t, tid.encode(), out.ctypes.data_as(C.c_void_p), out.nbytes):
        _err()
    return out


def map_eval_all(map_json: dict):
    """(sorted target names, target index, offset) of a reference IndexMap over its domain."""
    shape = map_json["virtual_shape"]
    n = int(np.prod(shape)) if shape else 1
    t = np.empty(n, np.int32)
    o = np.empty(n, np.int64)
    if lib().vref_map_eval_all(json.dumps(map_json).encode(), t.ctypes.data_as(C.POINTER(C.c_int32)),
                               o.ctypes.data_as(C.POINTER(C.c_int64)), n):
        _err()
    targets = sorted({p["target"] for p in map_json["pieces"]})
    return targets, t, o


def map_analyze(map_json: dict, elem_size: int = 4, coalesce: int = 128) -> dict:
    s = lib().vref_map_analyze(json.dumps(map_json).encode(), elem_size, coalesce)
    if s is None:
        _err()
    return json.loads(s.decode())

"""Python mirror of the reference's executor-facing API over the C ABI.

Names and argument meaning follow the reference (vtelim):
  parse_graph(text) -> CompGraph              proj/src/graph_ir.cpp:455-485
  CompGraph.vtog()                             build_vtog, proj/src/vtog.cpp:31-78
  Plan(graph, mode, selected)                  all_physical_ptg / validate_ptg
  execute(graph, plan, inputs) -> outputs      proj/src/executor.cpp:500-506
and errors are raised as the reference's error classes
(proj/include/vtelim/errors.hpp:14-38).  Host arrays are numpy; bf16 tensors
travel as uint16 bit patterns.  All compute runs in libvtc.so on the GPU.
"""
from __future__ import annotations

import ctypes as C
import json
from typing import Dict, Iterable, Optional, Sequence

import numpy as np

from . import _lib


class VtcError(RuntimeError):
    code = 1


_ERROR_NAMES = {
    2: "SchemaError", 3: "CycleError", 4: "ShapeError", 5: "UnknownOperatorError",
    6: "OutOfBoundsError", 7: "MissingBaseMapError", 8: "ComposeLimitError",
    9: "ConflictViolationError", 10: "IncompleteSelectionError", 11: "CycleDetectedError",
    12: "WriteAliasingError", 13: "SpaceTooLargeError", 14: "MissingInputError",
    15: "ShapeMismatchError", 16: "ExecutionError", 17: "EquivalenceFailureError",
    18: "InvalidVtogError", 19: "BudgetExceededError", 20: "CudaError", 21: "NcclError",
    22: "UnsupportedError",
}
ERRORS = {code: type(name, (VtcError,), {"code": code}) for code, name in _ERROR_NAMES.items()}
globals().update({cls.__name__: cls for cls in ERRORS.values()})

MATERIALIZE, SELECTED, MAX_ELIMINATION, INPLACE_UPDATES, GREEDY = 0, 1, 2, 3, 4
FLAG_FAST_FP, FLAG_NO_GEMV, FLAG_NO_FUSE, FLAG_GEMV_LDG, FLAG_NO_TC, FLAG_DYNAMIC_POS = 1, 2, 4, 8, 16, 32

NP_DTYPES = {"f64": np.float64, "f32": np.float32, "i64": np.int64, "bf16": np.uint16}


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib.load().vtc_last_error().decode()
        raise ERRORS.get(rc, VtcError)(msg)


def _stream(s) -> C.c_void_p:
    if s is None:
        return C.c_void_p(0)
    if isinstance(s, int):
        return C.c_void_p(s)
    return C.c_void_p(int(s.cuda_stream))  # torch.cuda.Stream


class CompGraph:
    def __init__(self, handle: C.c_void_p, text: str):
        self._h = handle
        self.text = text
        self.doc = json.loads(text)
        self._specs = None

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                _lib.load().vtc_graph_free(self._h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    def serialize(self) -> str:
        out = C.c_char_p()
        _check(_lib.load().vtc_graph_serialize(self._h, C.byref(out)))
        return out.value.decode()

    def tensors(self) -> Dict[str, dict]:
        if self._specs is None:
            doc = json.loads(self.serialize())
            self._specs = {t["id"]: t for t in doc["tensors"]}
        return self._specs

    def graph_inputs(self):
        return [k for k, t in self.tensors().items() if t["kind"] == "input"]

    def graph_outputs(self):
        return [k for k, t in self.tensors().items() if t["kind"] == "output"]

    def vtog(self) -> dict:
        out = C.c_char_p()
        _check(_lib.load().vtc_graph_vtog(self._h, C.byref(out)))
        return json.loads(out.value.decode())

    @staticmethod
    def _params(params) -> Optional[bytes]:
        if params is None:
            return None
        return (params if isinstance(params, str) else json.dumps(params)).encode()

    def estimate(self, selected: Optional[Iterable[int]] = None, params=None) -> dict:
        """vtelim::estimate(g, ptg, MachineParams) + breakdown; selected=None is the
        all-physical plan, params None = reference defaults, "b200" = calibrated."""
        out = C.c_char_p()
        if selected is None:
            arr, n = None, -1
        else:
            sel = list(selected)
            arr, n = (C.c_int32 * max(1, len(sel)))(*sel), len(sel)
        _check(_lib.load().vtc_graph_estimate(self._h, arr, n, self._params(params), C.byref(out)))
        return json.loads(out.value.decode())

    def saving(self, selected: Iterable[int], params=None) -> float:
        """The analytic SavingOracle: estimate(all-physical) - estimate(selected)."""
        return self.estimate(None, params)["total_time"] - self.estimate(selected, params)["total_time"]

    def enumerate_ptgs(self, limit: int = -1) -> list:
        out = C.c_char_p()
        _check(_lib.load().vtc_graph_enumerate(self._h, int(limit), C.byref(out)))
        return json.loads(out.value.decode())["ptgs"]

    def greedy(self, oracle: str = "analytic", params=None, trials: int = 5, executable: bool = False) -> dict:
        """Alg. 2 (global greedy) over the analytic or the B200-timed saving oracle."""
        cfg = {"oracle": oracle, "trials": trials, "executable": executable}
        if params is not None:
            cfg["params"] = params
        out = C.c_char_p()
        _check(_lib.load().vtc_graph_greedy(self._h, json.dumps(cfg).encode(), C.byref(out)))
        return json.loads(out.value.decode())


def parse_graph(text) -> CompGraph:
    if isinstance(text, dict):
        text = json.dumps(text)
    h = C.c_void_p()
    _check(_lib.load().vtc_graph_parse(text.encode(), C.byref(h)))
    return CompGraph(h, text)


_ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bit patterns (uint16)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + 0x7FFF
    out = ((u + r) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        out[nan] = 0x7FC0
    return out


class Comm:
    """NCCL communicator for tensor-parallel plans (include/vtc.h vtc_comm_*):
    rank 0 calls Comm.unique_id(), the id is shared over any host channel, every
    rank constructs Comm(uid, nranks, rank) on its current CUDA device."""

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_char * 128)()
        _check(_lib.load().vtc_comm_unique_id(C.cast(buf, C.c_void_p), 128))
        return bytes(buf)

    def __init__(self, uid: bytes, nranks: int, rank: int):
        assert len(uid) == 128
        h = C.c_void_p()
        buf = (C.c_char * 128).from_buffer_copy(uid)
        _check(_lib.load().vtc_comm_init(C.cast(buf, C.c_void_p), 128, nranks, rank, C.byref(h)))
        self._h = h
        self.nranks, self.rank = nranks, rank

    @classmethod
    def host_bridged(cls, allreduce, nranks: int, rank: int) -> "Comm":
        """A communicator whose AllReduce nodes stage through pinned host memory and
        call allreduce(values) -> summed values (a numpy array of the buffer's dtype,
        float32 for bf16 buffers, which are rounded back once) from a CUDA stream host
        node (include/vtc.h vtc_comm_init_host), e.g. torch.distributed over gloo."""
        self = cls.__new__(cls)
        dtypes = {0: np.float64, 1: np.float32, 2: np.int64, 3: np.uint16}

        def cb(_user, buf, count, dtype):
            try:
                n = int(count)
                raw = np.ctypeslib.as_array((C.c_byte * (n * np.dtype(dtypes[dtype]).itemsize)).from_address(buf))
                arr = raw.view(dtypes[dtype])
                if dtype == 3:
                    f32 = (arr.astype(np.uint32) << 16).view(np.float32)
                    arr[:] = f32_to_bf16_bits(np.asarray(allreduce(f32), dtype=np.float32))
                else:
                    arr[:] = np.asarray(allreduce(arr.copy()), dtype=arr.dtype)
                return 0
            except Exception:  # surfaced as a wrong result by the caller's checks
                import traceback
                traceback.print_exc()
                return 1

        self._cb = _ALLREDUCE_FN(cb)  # keep alive as long as the communicator
        h = C.c_void_p()
        _check(_lib.load().vtc_comm_init_host(C.cast(self._cb, C.c_void_p), None, nranks, rank, C.byref(h)))
        self._h = h
        self.nranks, self.rank = nranks, rank
        return self

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                _lib.load().vtc_comm_free(self._h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None


class Plan:
    """A points-to graph bound to the GPU executor (roots own device memory)."""

    def __init__(self, graph: CompGraph, mode: int = MAX_ELIMINATION, selected: Optional[Iterable[int]] = None,
                 flags: int = 0):
        self.graph = graph
        sel = list(selected or [])
        arr = (C.c_int32 * max(1, len(sel)))(*sel)
        h = C.c_void_p()
        _check(_lib.load().vtc_plan_create(graph._h, mode, arr, len(sel), flags, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                _lib.load().vtc_plan_free(self._h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    def info(self, dry: bool = False) -> dict:
        out = C.c_char_p()
        _check(_lib.load().vtc_plan_info(self._h, 1 if dry else 0, C.byref(out)))
        return json.loads(out.value.decode())

    def bind_root(self, tensor: str, dev_ptr: int) -> None:
        _check(_lib.load().vtc_plan_bind_root(self._h, tensor.encode(), C.c_void_p(dev_ptr)))

    def root_ptr(self, tensor: str) -> int:
        p = C.c_void_p()
        _check(_lib.load().vtc_plan_root_ptr(self._h, tensor.encode(), C.byref(p)))
        return p.value or 0

    def upload(self, tensor: str, arr: np.ndarray, stream=None) -> None:
        arr = np.ascontiguousarray(arr)
        _check(_lib.load().vtc_plan_upload(self._h, tensor.encode(), arr.ctypes.data_as(C.c_void_p),
                                           arr.nbytes, _stream(stream)))

    def upload_ptr(self, tensor: str, host_ptr: int, nbytes: int, stream=None) -> None:
        """H2D from a raw host pointer (e.g. pinned memory)."""
        _check(_lib.load().vtc_plan_upload(self._h, tensor.encode(), C.c_void_p(host_ptr), nbytes, _stream(stream)))

    def download_ptr(self, tensor: str, host_ptr: int, nbytes: int, stream=None) -> None:
        _check(_lib.load().vtc_plan_download(self._h, tensor.encode(), C.c_void_p(host_ptr), nbytes,
                                             _stream(stream)))

    def download(self, tensor: str, stream=None) -> np.ndarray:
        spec = self.graph.tensors()[tensor]
        out = np.empty(spec["shape"], dtype=NP_DTYPES[spec["dtype"]])
        _check(_lib.load().vtc_plan_download(self._h, tensor.encode(), out.ctypes.data_as(C.c_void_p),
                                             out.nbytes, _stream(stream)))
        return out

    def host_step(self, inputs, outputs, stream=None):
        """A bound vtc_run call for repeated steps from fixed host buffers:
        `inputs` / `outputs` are lists of (tensor id, host pointer, nbytes).
        The ctypes argument arrays are built once; calling the returned
        function runs one step (one H2D, graph replay, D2H, stream sync).
        Pinned host buffers make the copies asynchronous DMA."""
        ni, no = len(inputs), len(outputs)
        args = (self._h, ni,
                (C.c_char_p * max(ni, 1))(*[t.encode() for t, _, _ in inputs]),
                (C.c_void_p * max(ni, 1))(*[C.c_void_p(p) for _, p, _ in inputs]),
                (C.c_int64 * max(ni, 1))(*[n for _, _, n in inputs]),
                no,
                (C.c_char_p * max(no, 1))(*[t.encode() for t, _, _ in outputs]),
                (C.c_void_p * max(no, 1))(*[C.c_void_p(p) for _, p, _ in outputs]),
                (C.c_int64 * max(no, 1))(*[n for _, _, n in outputs]),
                _stream(stream))
        fn = _lib.load().vtc_run

        def step():
            rc = fn(*args)
            if rc:
                _check(rc)
        step._keep = (self, args)  # noqa: SLF001 -- keep the plan and buffers alive
        return step

    def run_ptrs(self, inputs, outputs, stream=None) -> None:
        """One step from host memory through vtc_run (see host_step)."""
        self.host_step(inputs, outputs, stream)()

    def run(self, inputs: Dict[str, np.ndarray], outputs: Sequence[str], stream=None) -> Dict[str, np.ndarray]:
        """execute(g, ptg, inputs) for one step: upload `inputs`, run, return `outputs`."""
        arrs = {k: np.ascontiguousarray(v) for k, v in inputs.items()}
        tens = self.graph.tensors()
        res = {o: np.empty(tens[o]["shape"], dtype=NP_DTYPES[tens[o]["dtype"]]) for o in outputs}
        self.run_ptrs([(k, a.ctypes.data, a.nbytes) for k, a in arrs.items()],
                      [(k, a.ctypes.data, a.nbytes) for k, a in res.items()], stream)
        return res

    def prepare(self) -> None:
        _check(_lib.load().vtc_plan_prepare(self._h))

    def set_position(self, pos: int, stream=None) -> None:
        """Dynamic-position plans (FLAG_DYNAMIC_POS): the next executions write
        cache row `pos` and attend over keys [0, pos].  vtc_run callers can pass
        the position as the input "__pos" (int64[1]) instead."""
        _check(_lib.load().vtc_plan_set_position(self._h, int(pos), _stream(stream)))

    def execute(self, stream=None) -> None:
        _check(_lib.load().vtc_execute(self._h, _stream(stream)))

    def execute_graph(self, stream=None) -> None:
        _check(_lib.load().vtc_execute_graph(self._h, _stream(stream)))

    def execute_timed(self, n_records: int, stream=None) -> np.ndarray:
        ms = np.zeros(max(1, n_records), np.float32)
        _check(_lib.load().vtc_execute_timed(self._h, _stream(stream), ms.ctypes.data_as(C.POINTER(C.c_float)),
                                             n_records))
        return ms

    def set_comm(self, comm: Optional["Comm"]) -> None:
        """Run this plan's AllReduce nodes on `comm` (None: single rank)."""
        self._comm = comm  # keep alive
        _check(_lib.load().vtc_plan_set_comm(self._h, comm._h if comm is not None else None))

    def trace(self) -> np.ndarray:
        """[n_launches, 8] globaltimer (ns): entry, exit, kernel checkpoints per
        launch since the last call (plans prepared with VTC_TRACE=1), else empty."""
        n = max(1, self.num_launches())
        buf = np.zeros(8 * n, np.uint64)
        r = _lib.load().vtc_plan_trace(self._h, buf.ctypes.data_as(C.POINTER(C.c_uint64)), 8 * n)
        if r < 0:
            _check(-r)
        return buf[: 8 * r].reshape(r, 8)

    def num_launches(self) -> int:
        return _lib.load().vtc_plan_num_launches(self._h)

    def map_json(self, tensor: str) -> dict:
        out = C.c_char_p()
        _check(_lib.load().vtc_plan_map_json(self._h, tensor.encode(), C.byref(out)))
        return json.loads(out.value.decode())

    def map_analyze(self, tensor: str, elem_size: int = 4, coalesce: int = 128) -> dict:
        out = C.c_char_p()
        _check(_lib.load().vtc_plan_map_analyze(self._h, tensor.encode(), elem_size, coalesce, C.byref(out)))
        return json.loads(out.value.decode())

    def map_eval(self, tensor: str, lowered: bool = False):
        """(target names, target index per element, offsets) in row-major order."""
        mj = self.map_json(tensor)
        n = int(np.prod(mj["shape"])) if mj["shape"] else 1
        t = np.empty(n, np.int32)
        o = np.empty(n, np.int64)
        _check(_lib.load().vtc_map_eval(self._h, tensor.encode(), 1 if lowered else 0,
                                        t.ctypes.data_as(C.POINTER(C.c_int32)),
                                        o.ctypes.data_as(C.POINTER(C.c_int64)), n))
        return mj["targets"], t, o


def execute(graph: CompGraph, plan: Plan, inputs: Dict[str, np.ndarray], roots: Iterable[str] = (),
            stream=None) -> Dict[str, np.ndarray]:
    """Reference `execute` semantics: upload inputs, run, materialise outputs (and requested roots)."""
    for name in graph.graph_inputs():
        if name not in inputs:
            raise ERRORS[14](f"input tensor {name} not provided")
        spec = graph.tensors()[name]
        a = inputs[name]
        if list(a.shape) != spec["shape"] or a.dtype != NP_DTYPES[spec["dtype"]]:
            raise ERRORS[15](f"input tensor {name} shape or dtype mismatch")
        plan.upload(name, a, stream)
    plan.execute(stream)
    out = {name: plan.download(name, stream) for name in graph.graph_outputs()}
    for r in roots:
        out["root:" + r] = plan.download(r, stream)
    return out


# ---- bf16 helpers (host) ----------------------------------------------------
def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bit patterns (uint16)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    lsb = (b >> 16) & 1
    r = ((b + 0x7FFF + lsb) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        r = np.where(nan, np.uint16(0x7FC0), r)
    return r


def bf16_to_f32(x: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(x, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)

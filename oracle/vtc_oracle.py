"""CPU oracle: numpy restatement of the reference interpreter's operator semantics.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
bench.py's cpu / reference legs as the *checker*; the product path
(paper_2604_09558_b200 / libvtc.so) never imports it.

Restates, operator by operator, proj/src/executor.cpp run_operator (:253-435):
  MatMul    :230-249  batched, acc in T, k ascending (f32/f64 bit-exact via a
                      k-sequential numpy loop; i64 wrapping)
  Add/Mul   :268-280  elementwise in T
  SiLU      :224-227, 281-291  computed in double, cast to T
  Transpose :292-311, Reshape/Unsqueeze :312-318, Split :319-343,
  Concat    :344-369, Slice :370-391, Expand :392-411 (x[i mod in_extent]),
  ScatterND :412-432 (clone + update slabs)
and execute (:448-506) on the all-physical plan (every tensor materialised;
by the reference's equivalence contract, any valid plan
gives the same outputs).  Pinned against oracle/_ref (the reference library
itself) in tests/test_oracle_pinning.py.

Extensions absent from the reference (SURVEY.md §8 a') -- parity for these is
unpinned by the reference; their semantics are fixed here and in the CUDA
kernels (k_rowop.cu, k_attention.cu): bf16 storage with RNE rounding after
every op (fp32 math), RMSNorm, LayerNorm, Softmax, GELU (erf), Attention
(softmax(scale*QK^T [+bias] [causal]) V), AllReduce (identity on one rank),
Roll (torch.roll).
"""
from __future__ import annotations

import json
import math
from typing import Dict

import numpy as np

NP = {"f64": np.float64, "f32": np.float32, "i64": np.int64, "bf16": np.uint16}


def f32_to_bf16(x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)
    return np.where(np.isnan(x), np.uint16(0x7FC0), r)


def bf16_to_f32(x):
    return (np.ascontiguousarray(x, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


class Graph:
    def __init__(self, doc):
        if isinstance(doc, str):
            doc = json.loads(doc)
        self.doc = doc
        self.tensors = {t["id"]: dict(t) for t in doc["tensors"]}
        self.nodes = doc["nodes"]
        self._infer()
        self.order = self._topo()

    def _topo(self):
        prod = {}
        for i, n in enumerate(self.nodes):
            for o in n["outputs"]:
                prod[o] = i
        waiting = [sum(1 for t in n["inputs"] if t in prod) for n in self.nodes]
        cons = {}
        for i, n in enumerate(self.nodes):
            for t in n["inputs"]:
                cons.setdefault(t, []).append(i)
        import heapq
        ready = [i for i, w in enumerate(waiting) if w == 0]
        heapq.heapify(ready)
        order = []
        while ready:
            i = heapq.heappop(ready)
            order.append(i)
            for o in self.nodes[i]["outputs"]:
                for c in cons.get(o, []):
                    waiting[c] -= 1
                    if waiting[c] == 0:
                        heapq.heappush(ready, c)
        assert len(order) == len(self.nodes), "cycle"
        return order

    def _infer(self):
        # shapes are produced by running shape rules lazily in execute(); the
        # JSON builders in workloads.py leave intermediate shapes empty.
        pass

    def inputs(self):
        return [t["id"] for t in self.doc["tensors"] if t["kind"] == "input"]

    def outputs(self):
        return [t["id"] for t in self.doc["tensors"] if t["kind"] == "output"]


def _to_compute(a, dt):
    return bf16_to_f32(a) if dt == "bf16" else a


def _from_compute(a, dt):
    if dt == "bf16":
        return f32_to_bf16(np.asarray(a, dtype=np.float32))
    return np.asarray(a).astype(NP[dt], copy=False)


def matmul_seq(a, b, dt):
    """Reference matmul_kernel: acc in T, k ascending (executor.cpp:238-247)."""
    if dt == "i64":
        with np.errstate(over="ignore"):
            acc = np.zeros(a.shape[:-1] + (b.shape[-1],), dtype=np.int64)
            for k in range(a.shape[-1]):
                acc = acc + a[..., :, k:k + 1] * b[..., k:k + 1, :]
            return acc
    if dt in ("f32", "f64"):
        t = NP[dt]
        acc = np.zeros(a.shape[:-1] + (b.shape[-1],), dtype=t)
        for k in range(a.shape[-1]):
            prod = (a[..., :, k:k + 1] * b[..., k:k + 1, :]).astype(t)
            acc = (acc + prod).astype(t)
        return acc
    # bf16 (extension): exact products, fp64 accumulation, one RNE rounding
    return f32_to_bf16(np.matmul(bf16_to_f32(a).astype(np.float64), bf16_to_f32(b).astype(np.float64)))


def run_operator(n, ins, dt, out_shapes=None):
    kind, at = n["kind"], n.get("attrs", {})
    if kind == "MatMul":
        return [matmul_seq(ins[0], ins[1], dt)]
    if kind in ("Add", "Mul"):
        x, y = _to_compute(ins[0], dt), _to_compute(ins[1], dt)
        with np.errstate(over="ignore"):
            z = x + y if kind == "Add" else x * y
        return [_from_compute(z, dt)]
    if kind == "SiLU":
        if dt == "bf16":
            x = bf16_to_f32(ins[0])
            return [f32_to_bf16((x / (np.float32(1) + np.exp(-x))).astype(np.float32))]
        x = ins[0].astype(np.float64)
        # libm exp (what std::exp calls) rather than numpy's SIMD exp, so the
        # restatement stays bit-identical to the reference for f32/f64
        e = np.frompyfunc(math.exp, 1, 1)(-x).astype(np.float64) if x.size <= (1 << 20) else np.exp(-x)
        return [(x / (1.0 + e)).astype(NP[dt])]
    if kind == "GELU":
        from scipy.special import erf
        x = _to_compute(ins[0], dt).astype(np.float64)
        return [_from_compute(0.5 * x * (1.0 + erf(x / math.sqrt(2.0))), dt)]
    if kind == "Transpose":
        return [np.ascontiguousarray(np.transpose(ins[0], at["perm"]))]
    if kind == "Reshape":
        return [ins[0].reshape(at["shape"]).copy()]
    if kind == "Unsqueeze":
        return [np.expand_dims(ins[0], at["axis"]).copy()]
    if kind == "Split":
        idx = np.cumsum(at["sizes"])[:-1]
        return [p.copy() for p in np.split(ins[0], idx, axis=at["axis"])]
    if kind == "Concat":
        return [np.concatenate(ins, axis=at["axis"])]
    if kind == "Slice":
        sl = [slice(None)] * ins[0].ndim
        for ax, s, e in zip(at["axes"], at["starts"], at["ends"]):
            sl[ax] = slice(s, e)
        return [ins[0][tuple(sl)].copy()]
    if kind == "Expand":
        reps = [o // i for o, i in zip(at["shape"], ins[0].shape)]
        return [np.tile(ins[0], reps)]
    if kind == "ScatterND":
        z = ins[0].copy()
        for m, tup in enumerate(at["indices"]):
            z[tuple(tup)] = ins[1][m]
        return [z]
    if kind == "Roll":
        return [np.roll(ins[0], at["shifts"], axis=at["axes"])]
    if kind == "AllReduce":
        return [ins[0].copy()]
    if kind in ("RMSNorm", "LayerNorm", "Softmax"):
        wide = np.float64 if dt == "f64" else np.float32
        x = _to_compute(ins[0], dt).astype(wide)
        eps = wide(at.get("eps", 1e-5))
        if kind == "RMSNorm":
            w = _to_compute(ins[1], dt).astype(wide)
            ms = np.mean(x.astype(np.float64) ** 2, axis=-1, keepdims=True).astype(wide)
            r = (1.0 / np.sqrt(ms + eps)).astype(wide)
            y = (x * r) * w
        elif kind == "LayerNorm":
            g, b = _to_compute(ins[1], dt).astype(wide), _to_compute(ins[2], dt).astype(wide)
            mu = np.mean(x.astype(np.float64), axis=-1, keepdims=True).astype(wide)
            var = np.mean((x - mu).astype(np.float64) ** 2, axis=-1, keepdims=True).astype(wide)
            y = ((x - mu) * (1.0 / np.sqrt(var + eps)).astype(wide)) * g + b
        else:
            mx = np.max(x, axis=-1, keepdims=True)
            e = np.exp(x - mx)
            y = e / np.sum(e.astype(np.float64), axis=-1, keepdims=True).astype(wide)
        return [_from_compute(y, dt)]
    if kind == "Attention":
        q, k, v = (_to_compute(t, dt).astype(np.float64) for t in ins[:3])
        s = np.matmul(q, np.swapaxes(k, -1, -2)) * at.get("scale", 1.0)
        if len(ins) == 4:
            s = s + _to_compute(ins[3], dt).astype(np.float64)
        if at.get("causal", False):
            sq, sk = s.shape[-2], s.shape[-1]
            mask = np.arange(sk)[None, :] > (np.arange(sq)[:, None] + (sk - sq))
            s = np.where(mask, -np.inf, s)
        s = s - np.max(s, axis=-1, keepdims=True)
        p = np.exp(s)
        p = p / np.sum(p, axis=-1, keepdims=True)
        return [_from_compute(np.matmul(p, v), dt)]
    raise ValueError(f"oracle: no semantics for operator {kind}")


def execute(doc, inputs: Dict[str, np.ndarray], keep_all: bool = False, allreduce=None) -> Dict[str, np.ndarray]:
    """All-physical execution (reference `execute`, executor.cpp:500-506).

    `allreduce(values_f32) -> summed_f32` performs a tensor-parallel AllReduce
    across ranks (e.g. torch.distributed over gloo in the multi-process tests);
    without it AllReduce is the single-rank identity.  bf16 partials are summed
    in fp32 and rounded once, like ncclAllReduce(ncclBfloat16) with two ranks."""
    g = doc if isinstance(doc, Graph) else Graph(doc)
    env = {}
    for tid in g.inputs():
        if tid not in inputs:
            raise KeyError(f"input tensor {tid} not provided")
        env[tid] = np.ascontiguousarray(inputs[tid])
    for i in g.order:
        n = g.nodes[i]
        dt = g.tensors[n["inputs"][0]]["dtype"]
        if n["kind"] == "AllReduce" and allreduce is not None:
            x = env[n["inputs"][0]]
            s = np.asarray(allreduce(_to_compute(x, dt).astype(np.float32)))
            env[n["outputs"][0]] = f32_to_bf16(s) if dt == "bf16" else s.astype(x.dtype)
            continue
        outs = run_operator(n, [env[t] for t in n["inputs"]], dt)
        for name, val in zip(n["outputs"], outs):
            env[name] = val
    if keep_all:
        return env
    return {t: env[t] for t in g.outputs()}


def random_inputs(doc, seed: int = 1, scales: Dict[str, float] | None = None) -> Dict[str, np.ndarray]:
    """Seeded uniform(-1, 1) inputs (i64: integers in [-8, 8]) in declaration order,
    scaled per tensor; bf16 tensors are rounded RNE.  Mirrors make_random_inputs'
    distribution (executor.cpp:508-528) with numpy's generator."""
    g = doc if isinstance(doc, Graph) else Graph(doc)
    rng = np.random.default_rng(seed)
    out = {}
    for tid in g.inputs():
        t = g.tensors[tid]
        shape = t["shape"]
        if t["dtype"] == "i64":
            out[tid] = rng.integers(-8, 9, size=shape, dtype=np.int64)
            continue
        x = rng.uniform(-1.0, 1.0, size=shape)
        if scales and tid in scales:
            x = x * scales[tid]
        if t["dtype"] == "bf16":
            out[tid] = f32_to_bf16(x.astype(np.float32))
        else:
            out[tid] = x.astype(NP[t["dtype"]])
    return out

"""Graph builders for the BASELINE.json workloads, in the reference JSON schema
(proj/src/graph_ir.cpp:455-485).

  c1_chain            configs[0]: reshape -> transpose -> slice feeding an fp32 matmul
  llama_decode_layer  configs[1]/[2]: Llama-3-8B decoder layer decode step with a
                      pos-major KV cache [S, B, Hkv, d] updated by ScatterND
  frame2_subgraph     the paper's Fig. 2 frame-2 chain (QKV -> KV-cache update -> QK)
                      in the reference's own operator vocabulary
Graphs are plain dicts; only reference operators plus the documented
extensions (RMSNorm, Attention, ...) are used.
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional


class GraphBuilder:
    def __init__(self, dtype: str = "f32"):
        self.dtype = dtype
        self.tensors: List[dict] = []
        self.nodes: List[dict] = []
        self._ids = set()

    def tensor(self, tid: str, shape=None, kind: str = "intermediate", dtype: Optional[str] = None) -> str:
        assert tid not in self._ids, tid
        self._ids.add(tid)
        t = {"id": tid, "dtype": dtype or self.dtype, "kind": kind}
        t["shape"] = list(shape) if shape is not None else []
        self.tensors.append(t)
        return tid

    def input(self, tid, shape, dtype=None):
        return self.tensor(tid, shape, "input", dtype)

    def node(self, nid: str, kind: str, inputs, outputs, attrs: Optional[dict] = None, out_kind: str = "intermediate"):
        outs = []
        for o in ([outputs] if isinstance(outputs, str) else outputs):
            if o not in self._ids:
                self.tensor(o, None, out_kind)
            outs.append(o)
        self.nodes.append({"id": nid, "kind": kind, "attrs": attrs or {}, "inputs": list(inputs), "outputs": outs})
        return outs[0] if len(outs) == 1 else outs

    def output(self, tid: str):
        for t in self.tensors:
            if t["id"] == tid:
                t["kind"] = "output"
        return tid

    def doc(self) -> dict:
        return {"tensors": self.tensors, "nodes": self.nodes}


def c1_chain(n: int = 1024, dtype: str = "f32") -> dict:
    """x [n,2,n] -> Reshape [n,2n] -> Transpose [2n,n] -> Slice rows [n/2, 3n/2) -> MatMul w [n,n].

    At n=1024 this is BASELINE configs[0]; s[m,k] = x_flat[n/2 + m + 2n*k].
    """
    g = GraphBuilder(dtype)
    g.input("x", [n, 2, n])
    g.input("w", [n, n])
    g.node("reshape", "Reshape", ["x"], "a", {"shape": [n, 2 * n]})
    g.node("transpose", "Transpose", ["a"], "t", {"perm": [1, 0]})
    g.node("slice", "Slice", ["t"], "s", {"axes": [0], "starts": [n // 2], "ends": [n // 2 + n]})
    g.node("matmul", "MatMul", ["s", "w"], "y", out_kind="output")
    return g.doc()


def llama_decode_layer(B: int = 1, L: int = 2048, pos: Optional[int] = None, D: int = 4096, Hq: int = 32,
                       Hkv: int = 8, hd: int = 128, F: int = 14336, dtype: str = "bf16", eps: float = 1e-5,
                       reference_ops_only: bool = False, tp: int = 1) -> dict:
    """One Llama-3 decoder layer, decode step (one new token per sequence).

    KV caches are pos-major [L, B, Hkv, hd] (the reference's ScatterND only
    supports 1-tuples, SURVEY.md §0 finding 1); the new token is written at
    `pos` and attention reads keys [0, pos].  RoPE uses the sign-folded
    rotate-half form  q*cos + concat(q[hd/2:], q[:hd/2])*sin_signed  so the
    rotation itself is a data-movement chain (Slice/Slice/Concat).
    reference_ops_only replaces RMSNorm by a weight Mul and Attention by
    MatMul(q, k^T) * scale -> MatMul(., v) (no softmax): the same data
    movement and the same GEMM work in the reference's vocabulary, used for
    the timed reference CPU arm.

    tp > 1 builds ONE rank's graph of a Megatron head-sharded layer
    (SURVEY.md §8 e): Hq/tp query heads, Hkv/tp KV heads and F/tp FFN columns
    are local (weights / caches are the rank's shards, see shard_llama_inputs),
    and exactly two AllReduce(sum) nodes -- after O-proj and after FFN-down --
    are the only exchange.  Every rank's graph is identical.
    """
    pos = L - 1 if pos is None else pos
    assert Hq % tp == 0 and Hkv % tp == 0 and F % tp == 0, "heads / FFN must divide the TP degree"
    Hq, Hkv, F = Hq // tp, Hkv // tp, F // tp
    G = Hq // Hkv
    half = hd // 2
    nq, nkv = Hq * hd, Hkv * hd
    g = GraphBuilder(dtype)
    g.input("x", [B, D])
    g.input("w_ln1", [D])
    g.input("w_qkv", [D, nq + 2 * nkv])
    g.input("cos", [B, hd])
    g.input("sin", [B, hd])
    g.input("k_cache", [L, B, Hkv, hd])
    g.input("v_cache", [L, B, Hkv, hd])
    g.input("w_o", [nq, D])
    g.input("w_ln2", [D])
    g.input("w_gate", [D, F])
    g.input("w_up", [D, F])
    g.input("w_down", [F, D])

    def norm(nid, x, w, out):
        if reference_ops_only:
            g.node(nid + "_wu", "Unsqueeze", [w], nid + "_w1", {"axis": 0})
            g.node(nid + "_we", "Expand", [nid + "_w1"], nid + "_wb", {"shape": [B, D]})
            return g.node(nid, "Mul", [x, nid + "_wb"], out)
        return g.node(nid, "RMSNorm", [x, w], out, {"eps": eps})

    norm("ln1", "x", "w_ln1", "h1")
    g.node("qkv_proj", "MatMul", ["h1", "w_qkv"], "qkv")
    g.node("qkv_split", "Split", ["qkv"], ["q2", "k2", "v2"], {"axis": 1, "sizes": [nq, nkv, nkv]})
    g.node("q_reshape", "Reshape", ["q2"], "q3", {"shape": [B, Hq, hd]})
    g.node("k_reshape", "Reshape", ["k2"], "k3", {"shape": [B, Hkv, hd]})
    g.node("v_reshape", "Reshape", ["v2"], "v3", {"shape": [B, Hkv, hd]})

    def rope(tag, x, H, out):
        g.node(f"{tag}_lo", "Slice", [x], f"{tag}_lo", {"axes": [2], "starts": [0], "ends": [half]})
        g.node(f"{tag}_hi", "Slice", [x], f"{tag}_hi", {"axes": [2], "starts": [half], "ends": [hd]})
        g.node(f"{tag}_rot", "Concat", [f"{tag}_hi", f"{tag}_lo"], f"{tag}_rot", {"axis": 2})
        for tab in ("cos", "sin"):
            g.node(f"{tag}_{tab}_u", "Unsqueeze", [tab], f"{tag}_{tab}_1", {"axis": 1})
            g.node(f"{tag}_{tab}_e", "Expand", [f"{tag}_{tab}_1"], f"{tag}_{tab}_b", {"shape": [B, H, hd]})
        g.node(f"{tag}_mc", "Mul", [x, f"{tag}_cos_b"], f"{tag}_xc")
        g.node(f"{tag}_ms", "Mul", [f"{tag}_rot", f"{tag}_sin_b"], f"{tag}_xs")
        return g.node(f"{tag}_add", "Add", [f"{tag}_xc", f"{tag}_xs"], out)

    rope("rq", "q3", Hq, "q_r")
    rope("rk", "k3", Hkv, "k_r")
    # KV-cache update at `pos` (ScatterND with static 1-tuples)
    g.node("k_unsq", "Unsqueeze", ["k_r"], "k_u", {"axis": 0})
    g.node("k_scatter", "ScatterND", ["k_cache", "k_u"], "kc2", {"indices": [[pos]]})
    g.node("v_unsq", "Unsqueeze", ["v3"], "v_u", {"axis": 0})
    g.node("v_scatter", "ScatterND", ["v_cache", "v_u"], "vc2", {"indices": [[pos]]})
    S = pos + 1

    def kv_path(tag, cache, out):
        src = cache
        if S < L:
            src = g.node(f"{tag}_slice", "Slice", [cache], f"{tag}_s", {"axes": [0], "starts": [0], "ends": [S]})
        g.node(f"{tag}_t", "Transpose", [src], f"{tag}_t", {"perm": [1, 2, 0, 3]})       # [B,Hkv,S,hd]
        g.node(f"{tag}_u", "Unsqueeze", [f"{tag}_t"], f"{tag}_u5", {"axis": 2})          # [B,Hkv,1,S,hd]
        g.node(f"{tag}_e", "Expand", [f"{tag}_u5"], f"{tag}_e", {"shape": [B, Hkv, G, S, hd]})
        return g.node(f"{tag}_r", "Reshape", [f"{tag}_e"], out, {"shape": [B, Hq, S, hd]})

    kv_path("kp", "kc2", "k_h")
    kv_path("vp", "vc2", "v_h")
    g.node("q_unsq", "Unsqueeze", ["q_r"], "q4", {"axis": 2})                         # [B,Hq,1,hd]
    scale = 1.0 / math.sqrt(hd)
    if reference_ops_only:
        g.node("k_tr", "Transpose", ["k_h"], "k_T", {"perm": [0, 1, 3, 2]})
        g.node("qk", "MatMul", ["q4", "k_T"], "sc")
        g.input("scale", [1, 1, 1, 1])
        g.node("sc_e", "Expand", ["scale"], "scale_b", {"shape": [B, Hq, 1, S]})
        g.node("sc_m", "Mul", ["sc", "scale_b"], "p")
        g.node("pv", "MatMul", ["p", "v_h"], "o4")
    else:
        g.node("attn", "Attention", ["q4", "k_h", "v_h"], "o4", {"scale": scale, "causal": False})
    g.node("o_reshape", "Reshape", ["o4"], "o2", {"shape": [B, nq]})
    if tp > 1:
        g.node("o_proj", "MatMul", ["o2", "w_o"], "ao_part")
        g.node("o_allreduce", "AllReduce", ["ao_part"], "ao")
    else:
        g.node("o_proj", "MatMul", ["o2", "w_o"], "ao")
    g.node("res1", "Add", ["x", "ao"], "x2")
    norm("ln2", "x2", "w_ln2", "h2")
    g.node("gate_proj", "MatMul", ["h2", "w_gate"], "gt")
    g.node("up_proj", "MatMul", ["h2", "w_up"], "up")
    g.node("silu", "SiLU", ["gt"], "sg")
    g.node("gate_mul", "Mul", ["sg", "up"], "mm")
    if tp > 1:
        g.node("down_proj", "MatMul", ["mm", "w_down"], "dn_part")
        g.node("down_allreduce", "AllReduce", ["dn_part"], "dn")
    else:
        g.node("down_proj", "MatMul", ["mm", "w_down"], "dn")
    g.node("res2", "Add", ["x2", "dn"], "y", out_kind="output")
    return g.doc()


def llama_prefill_layer(B: int = 8, S: int = 4096, D: int = 4096, Hq: int = 32, Hkv: int = 8, hd: int = 128,
                        F: int = 14336, dtype: str = "bf16", eps: float = 1e-5) -> dict:
    """One Llama-3 decoder layer over a prefill of S tokens per sequence
    (BASELINE configs[4]): T = B*S token rows, causal attention.  The QKV
    split, the RoPE rotate-half, the [B,S,H,d] <-> [B,H,S,d] transposes and the
    GQA Expand/Reshape of K/V are data-movement chains the planner turns into
    maps; the roped K and the V projection rows ([B,S,Hkv,d], token-major) are
    what a KV cache stores for these positions."""
    G = Hq // Hkv
    half = hd // 2
    nq, nkv = Hq * hd, Hkv * hd
    T = B * S
    g = GraphBuilder(dtype)
    g.input("x", [T, D])
    g.input("w_ln1", [D])
    g.input("w_qkv", [D, nq + 2 * nkv])
    g.input("cos", [B, S, hd])
    g.input("sin", [B, S, hd])
    g.input("w_o", [nq, D])
    g.input("w_ln2", [D])
    g.input("w_gate", [D, F])
    g.input("w_up", [D, F])
    g.input("w_down", [F, D])
    g.node("ln1", "RMSNorm", ["x", "w_ln1"], "h1", {"eps": eps})
    g.node("qkv_proj", "MatMul", ["h1", "w_qkv"], "qkv")
    g.node("qkv_split", "Split", ["qkv"], ["q2", "k2", "v2"], {"axis": 1, "sizes": [nq, nkv, nkv]})
    g.node("q_reshape", "Reshape", ["q2"], "q3", {"shape": [B, S, Hq, hd]})
    g.node("k_reshape", "Reshape", ["k2"], "k3", {"shape": [B, S, Hkv, hd]})
    g.node("v_reshape", "Reshape", ["v2"], "v3", {"shape": [B, S, Hkv, hd]})

    def rope(tag, x, H, out):
        g.node(f"{tag}_lo", "Slice", [x], f"{tag}_lo", {"axes": [3], "starts": [0], "ends": [half]})
        g.node(f"{tag}_hi", "Slice", [x], f"{tag}_hi", {"axes": [3], "starts": [half], "ends": [hd]})
        g.node(f"{tag}_rot", "Concat", [f"{tag}_hi", f"{tag}_lo"], f"{tag}_rot", {"axis": 3})
        for tab in ("cos", "sin"):
            g.node(f"{tag}_{tab}_u", "Unsqueeze", [tab], f"{tag}_{tab}_1", {"axis": 2})
            g.node(f"{tag}_{tab}_e", "Expand", [f"{tag}_{tab}_1"], f"{tag}_{tab}_b", {"shape": [B, S, H, hd]})
        g.node(f"{tag}_mc", "Mul", [x, f"{tag}_cos_b"], f"{tag}_xc")
        g.node(f"{tag}_ms", "Mul", [f"{tag}_rot", f"{tag}_sin_b"], f"{tag}_xs")
        return g.node(f"{tag}_add", "Add", [f"{tag}_xc", f"{tag}_xs"], out)

    rope("rq", "q3", Hq, "q_r")
    rope("rk", "k3", Hkv, "k_r")
    g.node("q_t", "Transpose", ["q_r"], "q4", {"perm": [0, 2, 1, 3]})

    def kv(tag, src, out):
        g.node(f"{tag}_t", "Transpose", [src], f"{tag}_t", {"perm": [0, 2, 1, 3]})           # [B,Hkv,S,hd]
        g.node(f"{tag}_u", "Unsqueeze", [f"{tag}_t"], f"{tag}_u5", {"axis": 2})
        g.node(f"{tag}_e", "Expand", [f"{tag}_u5"], f"{tag}_e", {"shape": [B, Hkv, G, S, hd]})
        return g.node(f"{tag}_r", "Reshape", [f"{tag}_e"], out, {"shape": [B, Hq, S, hd]})

    kv("kp", "k_r", "k_h")
    kv("vp", "v3", "v_h")
    g.node("attn", "Attention", ["q4", "k_h", "v_h"], "o4", {"scale": 1.0 / math.sqrt(hd), "causal": True})
    g.node("o_t", "Transpose", ["o4"], "o5", {"perm": [0, 2, 1, 3]})
    g.node("o_reshape", "Reshape", ["o5"], "o2", {"shape": [T, nq]})
    g.node("o_proj", "MatMul", ["o2", "w_o"], "ao")
    g.node("res1", "Add", ["x", "ao"], "x2")
    g.node("ln2", "RMSNorm", ["x2", "w_ln2"], "h2", {"eps": eps})
    g.node("gate_proj", "MatMul", ["h2", "w_gate"], "gt")
    g.node("up_proj", "MatMul", ["h2", "w_up"], "up")
    g.node("silu", "SiLU", ["gt"], "sg")
    g.node("gate_mul", "Mul", ["sg", "up"], "mm")
    g.node("down_proj", "MatMul", ["mm", "w_down"], "dn")
    g.node("res2", "Add", ["x2", "dn"], "y", out_kind="output")
    return g.doc()


def swin_block(B: int = 64, H: int = 56, C: int = 96, heads: int = 3, win: int = 7, shift: int = 3,
               mlp: int = 384, dtype: str = "bf16", eps: float = 1e-5) -> dict:
    """Swin-T stage-1 shifted-window transformer block (BASELINE configs[3]):
    x [B, H, H, C] -> LN -> cyclic Roll(-shift) -> window partition ->
    QKV linear -> W-MSA (relative-position bias + shift mask, one additive
    bias tensor per window) -> proj -> window reverse -> Roll(+shift) ->
    residual -> LN -> MLP (GELU) -> residual.  Roll, the partition / reverse
    reshapes and transposes, the QKV split and the per-window bias broadcast
    are data movement; under a VTC plan they are maps ((i + 3) mod 56,
    t div 7, t mod 7, ...) evaluated inside the LN / GEMM / attention kernels."""
    nw = (H // win) ** 2
    T = win * win
    hd = C // heads
    g = GraphBuilder(dtype)
    g.input("x", [B, H, H, C])
    g.input("ln1_g", [C])
    g.input("ln1_b", [C])
    g.input("w_qkv", [C, 3 * C])
    g.input("attn_bias", [nw, heads, T, T])   # relative-position bias + shift mask, per window
    g.input("w_proj", [C, C])
    g.input("ln2_g", [C])
    g.input("ln2_b", [C])
    g.input("w_fc1", [C, mlp])
    g.input("w_fc2", [mlp, C])
    g.node("ln1", "LayerNorm", ["x", "ln1_g", "ln1_b"], "xn", {"eps": eps})
    g.node("roll", "Roll", ["xn"], "xs", {"axes": [1, 2], "shifts": [-shift, -shift]})
    # window partition: [B, H/w, w, H/w, w, C] -> [B, H/w, H/w, w, w, C] -> [B*nw*T, C]
    g.node("part_r", "Reshape", ["xs"], "xp6", {"shape": [B, H // win, win, H // win, win, C]})
    g.node("part_t", "Transpose", ["xp6"], "xw6", {"perm": [0, 1, 3, 2, 4, 5]})
    g.node("part_f", "Reshape", ["xw6"], "xw", {"shape": [B * nw * T, C]})
    g.node("qkv_proj", "MatMul", ["xw", "w_qkv"], "qkv")
    g.node("qkv_r", "Reshape", ["qkv"], "qkv5", {"shape": [B * nw, T, 3, heads, hd]})
    g.node("qkv_t", "Transpose", ["qkv5"], "qkvt", {"perm": [2, 0, 3, 1, 4]})      # [3, B*nw, heads, T, hd]
    g.node("qkv_s", "Split", ["qkvt"], ["q5", "k5", "v5"], {"axis": 0, "sizes": [1, 1, 1]})
    for c in ("q", "k", "v"):
        g.node(f"{c}_r", "Reshape", [f"{c}5"], f"{c}4", {"shape": [B * nw, heads, T, hd]})
    g.node("bias_u", "Unsqueeze", ["attn_bias"], "bias5", {"axis": 0})                  # [1, nw, heads, T, T]
    g.node("bias_e", "Expand", ["bias5"], "bias_be", {"shape": [B, nw, heads, T, T]})
    g.node("bias_r", "Reshape", ["bias_be"], "bias4", {"shape": [B * nw, heads, T, T]})
    g.node("attn", "Attention", ["q4", "k4", "v4", "bias4"], "o4", {"scale": 1.0 / math.sqrt(hd), "causal": False})
    g.node("o_t", "Transpose", ["o4"], "o5", {"perm": [0, 2, 1, 3]})                     # [B*nw, T, heads, hd]
    g.node("o_r", "Reshape", ["o5"], "o2", {"shape": [B * nw * T, C]})
    g.node("proj", "MatMul", ["o2", "w_proj"], "pw")
    # window reverse + reverse roll
    g.node("rev_r", "Reshape", ["pw"], "pr6", {"shape": [B, H // win, H // win, win, win, C]})
    g.node("rev_t", "Transpose", ["pr6"], "pt6", {"perm": [0, 1, 3, 2, 4, 5]})
    g.node("rev_f", "Reshape", ["pt6"], "ps", {"shape": [B, H, H, C]})
    g.node("unroll", "Roll", ["ps"], "pu", {"axes": [1, 2], "shifts": [shift, shift]})
    g.node("res1", "Add", ["x", "pu"], "x2")
    g.node("ln2", "LayerNorm", ["x2", "ln2_g", "ln2_b"], "xn2", {"eps": eps})
    g.node("mlp_f", "Reshape", ["xn2"], "xm", {"shape": [B * H * H, C]})
    g.node("fc1", "MatMul", ["xm", "w_fc1"], "h1")
    g.node("gelu", "GELU", ["h1"], "h1g")
    g.node("fc2", "MatMul", ["h1g", "w_fc2"], "h2")
    g.node("mlp_b", "Reshape", ["h2"], "h2r", {"shape": [B, H, H, C]})
    g.node("res2", "Add", ["x2", "h2r"], "y", out_kind="output")
    return g.doc()


def c3k2_block(N: int = 16 * 160 * 160, c: int = 64, cin: int = 128, cout: int = 128, dtype: str = "bf16") -> dict:
    """Paper Fig. 11 (SPEC.md acceptance 7): the YOLOv11
    C3K2 block's data movement, channel-last with its 1x1 convolutions as
    MatMuls over the N = B*H*W pixels:

        y0 = x . W_cv1 -> Split(a, b) -> bottleneck on b: e = b + (SiLU(b . W_m1) . W_m2)
        Y  = Concat(a, b, e) -> out = Y . W_cv2

    Split and Concat are the block's two data-movement operators; under a VTC
    plan a, b and e (and y0) become virtual tensors of Y -- cv1 and the
    bottleneck's residual Add store straight into Y's channel ranges -- and no
    data-movement kernel runs."""
    g = GraphBuilder(dtype)
    g.input("x", [N, cin])
    g.input("w_cv1", [cin, 2 * c])
    g.input("w_m1", [c, c])
    g.input("w_m2", [c, c])
    g.input("w_cv2", [3 * c, cout])
    g.node("cv1", "MatMul", ["x", "w_cv1"], "y0")
    g.node("split", "Split", ["y0"], ["a", "b"], {"axis": 1, "sizes": [c, c]})
    g.node("m1", "MatMul", ["b", "w_m1"], "t1")
    g.node("act", "SiLU", ["t1"], "t2")
    g.node("m2", "MatMul", ["t2", "w_m2"], "t3")
    g.node("res", "Add", ["b", "t3"], "e")
    g.node("concat", "Concat", ["a", "b", "e"], "Y", {"axis": 1})
    g.node("cv2", "MatMul", ["Y", "w_cv2"], "out", out_kind="output")
    return g.doc()


def swin_attn_bias(H: int = 56, heads: int = 3, win: int = 7, shift: int = 3, seed: int = 0):
    """Per-window additive attention bias [nw, heads, T, T]: a random relative-
    position bias table gathered by relative coordinates (as in Swin) plus the
    -100 shift mask between tokens from different regions of a shifted window."""
    import numpy as np
    rng = np.random.default_rng(seed)
    table = rng.uniform(-0.1, 0.1, size=((2 * win - 1) ** 2, heads)).astype(np.float32)
    coords = np.stack(np.meshgrid(np.arange(win), np.arange(win), indexing="ij")).reshape(2, -1)
    rel = coords[:, :, None] - coords[:, None, :] + win - 1
    idx = rel[0] * (2 * win - 1) + rel[1]
    rpb = table[idx.reshape(-1)].reshape(win * win, win * win, heads).transpose(2, 0, 1)
    img = np.zeros((H, H), np.int32)
    cnt = 0
    for hs in (slice(0, -win), slice(-win, -shift), slice(-shift, None)):
        for ws in (slice(0, -win), slice(-win, -shift), slice(-shift, None)):
            img[hs, ws] = cnt
            cnt += 1
    nwin = H // win
    win_ids = img.reshape(nwin, win, nwin, win).transpose(0, 2, 1, 3).reshape(nwin * nwin, win * win)
    mask = np.where(win_ids[:, :, None] != win_ids[:, None, :], -100.0, 0.0).astype(np.float32)
    return (rpb[None, :, :, :] + mask[:, None, :, :]).astype(np.float32)


def swin_weight_scales(C: int = 96, mlp: int = 384) -> Dict[str, float]:
    return {"w_qkv": 1 / math.sqrt(C), "w_proj": 1 / math.sqrt(C), "w_fc1": 1 / math.sqrt(C),
            "w_fc2": 1 / math.sqrt(mlp), "ln1_g": 1.0, "ln2_g": 1.0, "ln1_b": 0.1, "ln2_b": 0.1}


def rope_tables_prefill(B: int, S: int, hd: int = 128, theta: float = 500000.0):
    """cos and sign-folded sin tables [B, S, hd] for positions 0..S-1."""
    import numpy as np
    cos, sin = rope_tables(S, list(range(S)), hd, theta)
    return np.broadcast_to(cos, (B, S, hd)).copy(), np.broadcast_to(sin, (B, S, hd)).copy()


def shard_llama_inputs(full: Dict, rank: int, tp: int, Hq: int = 32, Hkv: int = 8, hd: int = 128,
                       F: int = 14336) -> Dict:
    """Rank `rank`'s inputs of llama_decode_layer(tp=tp) from the full layer's
    inputs: Q/K/V columns and O rows of the local heads, gate/up columns and
    down rows of the local FFN slice, the local KV-cache heads; x, norms and
    RoPE tables replicated."""
    import numpy as np
    hq, hk, f = Hq // tp, Hkv // tp, F // tp
    nq, nkv = Hq * hd, Hkv * hd
    q_cols = np.arange(rank * hq * hd, (rank + 1) * hq * hd)
    k_cols = nq + np.arange(rank * hk * hd, (rank + 1) * hk * hd)
    v_cols = nq + nkv + np.arange(rank * hk * hd, (rank + 1) * hk * hd)
    out = dict(full)
    out["w_qkv"] = np.ascontiguousarray(full["w_qkv"][:, np.concatenate([q_cols, k_cols, v_cols])])
    out["w_o"] = np.ascontiguousarray(full["w_o"][q_cols, :])
    out["w_gate"] = np.ascontiguousarray(full["w_gate"][:, rank * f:(rank + 1) * f])
    out["w_up"] = np.ascontiguousarray(full["w_up"][:, rank * f:(rank + 1) * f])
    out["w_down"] = np.ascontiguousarray(full["w_down"][rank * f:(rank + 1) * f, :])
    for c in ("k_cache", "v_cache"):
        out[c] = np.ascontiguousarray(full[c][:, :, rank * hk:(rank + 1) * hk, :])
    return out


def llama_weight_scales(D: int = 4096, F: int = 14336) -> Dict[str, float]:
    """1/sqrt(fan_in) scaling applied to uniform(-1,1) weights (SURVEY.md §8 d)."""
    return {"w_qkv": 1 / math.sqrt(D), "w_o": 1 / math.sqrt(D), "w_gate": 1 / math.sqrt(D),
            "w_up": 1 / math.sqrt(D), "w_down": 1 / math.sqrt(F), "w_ln1": 1.0, "w_ln2": 1.0}


def rope_tables(B: int, positions, hd: int = 128, theta: float = 500000.0):
    """cos and sign-folded sin tables [B, hd] for the rotate-half RoPE form."""
    import numpy as np
    half = hd // 2
    inv = theta ** (-np.arange(half, dtype=np.float64) * 2.0 / hd)
    pos = np.asarray(positions, dtype=np.float64).reshape(B, 1)
    ang = pos * inv[None, :]
    cos = np.concatenate([np.cos(ang), np.cos(ang)], axis=1)
    sin = np.concatenate([-np.sin(ang), np.sin(ang)], axis=1)
    return cos, sin


def frame2_subgraph(B: int = 1, L: int = 64, pos: Optional[int] = None, D: int = 64, Hq: int = 4, Hkv: int = 1,
                    hd: int = 8, dtype: str = "f32") -> dict:
    """Paper Fig. 2 frame 2 in reference ops: QKV proj -> Split -> Reshape ->
    ScatterND(KV cache) -> Slice -> Transpose -> Unsqueeze -> Expand -> Reshape -> QK MatMul."""
    doc = llama_decode_layer(B=B, L=L, pos=pos, D=D, Hq=Hq, Hkv=Hkv, hd=hd, F=2 * D, dtype=dtype,
                             reference_ops_only=True)
    keep_nodes = []
    wanted = {"ln1_wu", "ln1_we", "ln1", "qkv_proj", "qkv_split", "q_reshape", "k_reshape", "v_reshape",
              "k_unsq", "k_scatter", "v_unsq", "v_scatter", "kp_slice", "kp_t", "kp_u", "kp_e", "kp_r",
              "vp_slice", "vp_t", "vp_u", "vp_e", "vp_r", "q_unsq", "k_tr", "qk", "sc_e", "sc_m", "pv"}
    for n in doc["nodes"]:
        if n["id"] in wanted:
            keep_nodes.append(n)
    # q_unsq reads q_r (rope output); rewire to q3 so the subgraph has no RoPE
    for n in keep_nodes:
        if n["id"] == "q_unsq":
            n["inputs"] = ["q3"]
        if n["id"] == "k_unsq":
            n["inputs"] = ["k3"]
    used = set()
    for n in keep_nodes:
        used.update(n["inputs"])
        used.update(n["outputs"])
    tensors = [dict(t) for t in doc["tensors"] if t["id"] in used]
    for t in tensors:
        if t["id"] == "o4":
            t["kind"] = "output"
        elif t["kind"] == "output":
            t["kind"] = "intermediate"
    return {"tensors": tensors, "nodes": keep_nodes}


# ---- paper-figure fixtures (acceptance 1-3, 7) -------------------
# Desk-scale graphs in the reference operator vocabulary only, so the
# reference planner / executor (oracle/_ref) runs every one of them.

def fig2_llama_subgraph(dtype: str = "f64") -> dict:
    """PAPER.md Fig. 2 frame 2 at the SPEC.md:478 size (B=2, heads=4, kv-heads=1,
    head-dim=8, ctx=16): QKV -> Split -> Reshape -> ScatterND(KV cache) -> Slice ->
    Transpose -> Unsqueeze -> Expand -> Reshape -> attention MatMuls."""
    return frame2_subgraph(B=2, L=16, pos=15, D=32, Hq=4, Hkv=1, hd=8, dtype=dtype)


def fig6_kv_update(dtype: str = "f64", L: int = 4, heads: int = 2, hd: int = 4, pos: int = 1) -> dict:
    """PAPER.md Fig. 6(a): MatMul -> Split -> Reshape -> ScatterND over the K cache.
    a = x.W; Split(a) -> (b, rest); c = Reshape(b); d = ScatterND(K cache, c @ pos).
    The Split's other output `rest` is a graph output ("other outputs of Split
    are ignored" in the figure); d feeds a scores MatMul so the cache is read."""
    D = heads * hd
    g = GraphBuilder(dtype)
    g.input("x", [1, D])
    g.input("W", [D, 3 * D])
    g.input("K_cache", [L, heads, hd])
    g.input("q", [heads, 1, hd])
    g.node("matmul", "MatMul", ["x", "W"], "a")
    g.node("split", "Split", ["a"], ["b", "rest"], {"axis": 1, "sizes": [D, 2 * D]})
    g.output("rest")
    g.node("reshape", "Reshape", ["b"], "c", {"shape": [1, heads, hd]})
    g.node("scatter", "ScatterND", ["K_cache", "c"], "d", {"indices": [[pos]]})
    g.node("kt", "Transpose", ["d"], "kT", {"perm": [1, 2, 0]})           # [heads, hd, L]
    g.node("scores", "MatMul", ["q", "kT"], "s", out_kind="output")       # [heads, 1, L]
    return g.doc()


def fig7_conflict(dtype: str = "f64", n: int = 4, m: int = 3) -> dict:
    """PAPER.md Fig. 7: c = Concat(a, b) and d = Transpose(c).  c's out-edges:
    1 = c over a, 2 = c over b (one Concat candidate: compatible), 3 = c over d
    (the Transpose read back): 1/3 and 2/3 conflict."""
    g = GraphBuilder(dtype)
    g.input("a", [n, m])
    g.input("b", [n, m])
    g.input("w", [n, 2])
    g.node("concat", "Concat", ["a", "b"], "c", {"axis": 1})             # [n, 2m]
    g.node("transpose", "Transpose", ["c"], "d", {"perm": [1, 0]})       # [2m, n]
    g.node("mm", "MatMul", ["d", "w"], "y", out_kind="output")
    return g.doc()


def fig9_efficientvit_attention(dtype: str = "f64", B: int = 2, N: int = 16, C: int = 16, heads: int = 2) -> dict:
    """PAPER.md Fig. 9 (EfficientViT linear-attention block): five
    compute kernels k1..k5 (qkv projection, K^T.V, Q.(K^T V), the output
    activation, the output projection); every data-movement operator between
    them is eliminable, leaving a (k1 out), e (k2 out), f (k3 out) and j (k4 out)
    as the only physical intermediates."""
    d = C // heads
    g = GraphBuilder(dtype)
    g.input("x", [B * N, C])
    g.input("W_qkv", [C, 3 * C])
    g.input("W_o", [C, C])
    g.node("k1", "MatMul", ["x", "W_qkv"], "a")                                   # [B*N, 3C]
    g.node("split", "Split", ["a"], ["q2", "k2", "v2"], {"axis": 1, "sizes": [C, C, C]})
    for t in ("q", "k", "v"):
        g.node(f"{t}_rs", "Reshape", [f"{t}2"], f"{t}4", {"shape": [B, N, heads, d]})
        g.node(f"{t}_tr", "Transpose", [f"{t}4"], f"{t}h", {"perm": [0, 2, 1, 3]})  # [B, H, N, d]
    g.node("kT", "Transpose", ["kh"], "kt", {"perm": [0, 1, 3, 2]})               # [B, H, d, N]
    g.node("k2_", "MatMul", ["kt", "vh"], "e")                                    # k2: [B, H, d, d]
    g.node("k3", "MatMul", ["qh", "e"], "f")                                      # k3: [B, H, N, d]
    g.node("f_tr", "Transpose", ["f"], "g", {"perm": [0, 2, 1, 3]})               # [B, N, H, d]
    g.node("g_rs", "Reshape", ["g"], "h", {"shape": [B * N, C]})
    g.node("k4", "SiLU", ["h"], "j")                                              # k4
    g.node("k5", "MatMul", ["j", "W_o"], "y", out_kind="output")                  # k5
    return g.doc()


def fig11_yolo_c3k2(dtype: str = "f64", N: int = 64, c: int = 4, cin: int = 8, cout: int = 8) -> dict:
    """PAPER.md Fig. 11 at desk scale in the paper's channel-first (NCHW) layout,
    so Split / Concat along channels move contiguous chunks of N pixels
    ("each contiguous chunk ... is large enough"); 1x1
    convolutions are W . X MatMuls over [channels, N]."""
    g = GraphBuilder(dtype)
    g.input("x", [cin, N])
    g.input("w_cv1", [2 * c, cin])
    g.input("w_m1", [c, c])
    g.input("w_m2", [c, c])
    g.input("w_cv2", [cout, 3 * c])
    g.node("cv1", "MatMul", ["w_cv1", "x"], "y0")
    g.node("split", "Split", ["y0"], ["a", "b"], {"axis": 0, "sizes": [c, c]})
    g.node("m1", "MatMul", ["w_m1", "b"], "t1")
    g.node("act", "SiLU", ["t1"], "t2")
    g.node("m2", "MatMul", ["w_m2", "t2"], "t3")
    g.node("res", "Add", ["b", "t3"], "e")
    g.node("concat", "Concat", ["a", "b", "e"], "Y", {"axis": 0})
    g.node("cv2", "MatMul", ["w_cv2", "Y"], "out", out_kind="output")
    return g.doc()


def chain_graph(n_tensors: int, dtype: str = "f64") -> dict:
    """A data-movement chain with `n_tensors` tensors (acceptance 6: greedy
    complexity): x -> (Transpose | Reshape)* -> MatMul."""
    g = GraphBuilder(dtype)
    g.input("x", [4, 6])
    g.input("w", [6, 3])
    cur, shape = "x", [4, 6]
    k = 0
    while len(g.tensors) < n_tensors - 1:
        k += 1
        out = f"t{k}"
        if k % 2:
            shape = shape[::-1]
            g.node(f"n{k}", "Transpose", [cur], out, {"perm": [1, 0]})
        else:
            g.node(f"n{k}", "Reshape", [cur], out, {"shape": list(shape)})
        cur = out
    if shape != [4, 6]:
        k += 1
        g.node(f"n{k}", "Transpose", [cur], f"t{k}", {"perm": [1, 0]})
        cur = f"t{k}"
    g.node("mm", "MatMul", [cur, "w"], "y", out_kind="output")
    return g.doc()

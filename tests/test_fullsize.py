"""Full-size parity of the benchmarked configurations (BASELINE.json configs[2..4])
on B200, checked against the CPU oracle on independent slices.

The product runs the exact bench workload (same graph builder, same sizes, so
the same launch list and kernel variants as bench.py); the oracle recomputes a
few independent units of it:

* C3 Llama-3-8B decode, B=64, KV 8192: batch rows are independent, so row b of
  y (and the KV-cache row written at pos for batch b) equals a B=1 oracle run
  on that row's x / RoPE row / KV-cache slice.
* C4 Swin-T block, B=64, 56x56: images are independent -> B=1 oracle runs.
* C5 Llama-3-8B prefill, B=8, S=4096: sequences are independent, and query row
  t of a sequence depends on rows 0..t only; the oracle evaluates the layer
  for rows {0, 1, 2047, 4095} of two sequences with the oracle's own
  operators (vtc_oracle.run_operator: the same per-op bf16 rounding), K / V
  projected for the whole causal prefix.

Tolerance: north-star bf16 bound, max |got - want| / max |want| < 2e-2.
Inputs are random bf16 (uniform(-1, 1), weights scaled by 1/sqrt(fan_in)).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _relerr(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want)) / max(1e-30, float(np.max(np.abs(want)))))


def _rand_bf16(rng, shape, scale=1.0):
    """Uniform(-scale, scale) bf16 bit patterns (truncated from float32: fast at GB sizes)."""
    x = rng.random(int(np.prod(shape)), dtype=np.float32)
    x *= np.float32(2 * scale)
    x -= np.float32(scale)
    return (x.view(np.uint32) >> 16).astype(np.uint16).reshape(shape)


def _inputs(doc, rng, scales, special=None):
    out = {}
    for t in doc["tensors"]:
        if t["kind"] != "input":
            continue
        if special and t["id"] in special:
            out[t["id"]] = special[t["id"]]
            continue
        out[t["id"]] = _rand_bf16(rng, t["shape"], scales.get(t["id"], 1.0))
    return out


def _kernels(plan):
    return [l["kernel"] for l in plan.info(dry=True)["launches"]]


def test_c3_decode_b64_kv8192_full_size(vtc, oracle):
    from paper_2604_09558_b200 import workloads as W
    B, L = 64, 8192
    pos = L - 1
    doc = W.llama_decode_layer(B=B, L=L)
    rng = np.random.default_rng(31)
    cos, sin = W.rope_tables(B, [pos] * B)
    x = _inputs(doc, rng, W.llama_weight_scales(),
                {"cos": oracle.f32_to_bf16(cos.astype(np.float32)), "sin": oracle.f32_to_bf16(sin.astype(np.float32))})
    g = vtc.parse_graph(doc)
    p = vtc.Plan(g, vtc.MAX_ELIMINATION)
    kinds = _kernels(p)
    assert p.info()["data_movement_launches"] == 0
    assert kinds.count("gemm_tc_bf16") >= 3 and "attn_decode_tc_splitkv" in kinds, kinds
    got = vtc.execute(g, p, x)["y"]
    kc = p.download("k_cache")
    vc = p.download("v_cache")
    doc1 = W.llama_decode_layer(B=1, L=L)
    errs = []
    for b in (0, 37):
        x1 = {k: v for k, v in x.items()}
        for k in ("x", "cos", "sin"):
            x1[k] = np.ascontiguousarray(x[k][b:b + 1])
        for k in ("k_cache", "v_cache"):
            x1[k] = np.ascontiguousarray(x[k][:, b:b + 1])
        env = oracle.execute(doc1, x1, keep_all=True)
        errs.append(_relerr(oracle.bf16_to_f32(got[b]), oracle.bf16_to_f32(env["y"][0])))
        # the new token's K (roped) / V rows were written in place at pos (fp32-accumulated
        # GEMM vs the oracle's fp64: equal up to the final bf16 rounding); other rows untouched
        for got_row, want_row in ((kc[pos, b], env["k_r"][0]), (vc[pos, b], env["v3"][0])):
            errs.append(_relerr(oracle.bf16_to_f32(got_row), oracle.bf16_to_f32(want_row)))
        assert np.array_equal(kc[:pos, b], x["k_cache"][:pos, b])
        assert np.array_equal(vc[:pos, b], x["v_cache"][:pos, b])
    print(f"C3 full size: rel err (y, K row, V row) per batch row {errs}")
    assert max(errs) < 2e-2, errs


def test_c4_swin_block_b64_full_size(vtc, oracle):
    from paper_2604_09558_b200 import workloads as W
    B, H = 64, 56
    doc = W.swin_block(B=B, H=H)
    rng = np.random.default_rng(41)
    bias = oracle.f32_to_bf16(W.swin_attn_bias())
    x = _inputs(doc, rng, W.swin_weight_scales(), {"attn_bias": bias})
    g = vtc.parse_graph(doc)
    p = vtc.Plan(g, vtc.MAX_ELIMINATION)
    kinds = _kernels(p)
    assert p.info()["data_movement_launches"] == 0
    assert kinds.count("gemm_skinny_bf16") == 4, kinds  # QKV (row gathers), proj, fc1 + GELU, fc2 + residual
    assert "attn_window_tc" in kinds, kinds  # one warp per (window, head)
    got = vtc.execute(g, p, x)["y"]
    doc1 = W.swin_block(B=1, H=H)
    errs = []
    for b in (0, 50):
        x1 = dict(x, x=np.ascontiguousarray(x["x"][b:b + 1]))
        want = oracle.execute(doc1, x1)["y"][0]
        errs.append(_relerr(oracle.bf16_to_f32(got[b]), oracle.bf16_to_f32(want)))
    print(f"C4 full size: max rel err per image {errs}")
    assert max(errs) < 2e-2, errs


def _op(oracle, kind, ins, **attrs):
    return oracle.run_operator({"kind": kind, "attrs": attrs}, ins, "bf16")[0]


def _prefill_rows_oracle(oracle, x, seq, rows, S, D=4096, Hq=32, Hkv=8, hd=128, eps=1e-5):
    """Rows `rows` of sequence `seq` of llama_prefill_layer's y, with the oracle's
    operators in the graph's order (causal attention over keys 0..t)."""
    G, half, nq, nkv = Hq // Hkv, hd // 2, Hq * hd, Hkv * hd
    xs = x["x"][seq * S:(seq + 1) * S]
    cos, sin = x["cos"][seq], x["sin"][seq]
    h1 = _op(oracle, "RMSNorm", [xs, x["w_ln1"]], eps=eps)
    wq = np.ascontiguousarray(x["w_qkv"][:, :nq])
    wkv = np.ascontiguousarray(x["w_qkv"][:, nq:])
    kv = _op(oracle, "MatMul", [h1, wkv])                       # [S, 2 nkv] (column subset of qkv)
    q = _op(oracle, "MatMul", [np.ascontiguousarray(h1[rows]), wq])

    def rope(t, c, s):
        rot = np.concatenate([t[..., half:], t[..., :half]], axis=-1)
        xc = _op(oracle, "Mul", [t, np.broadcast_to(c[:, None, :], t.shape)])
        xsn = _op(oracle, "Mul", [rot, np.broadcast_to(s[:, None, :], t.shape)])
        return _op(oracle, "Add", [xc, xsn])

    k_r = rope(kv[:, :nkv].reshape(S, Hkv, hd), cos, sin)
    v = kv[:, nkv:].reshape(S, Hkv, hd)
    q_r = rope(q.reshape(len(rows), Hq, hd), cos[rows], sin[rows])
    kf, vf = oracle.bf16_to_f32(k_r).astype(np.float64), oracle.bf16_to_f32(v).astype(np.float64)
    qf = oracle.bf16_to_f32(q_r).astype(np.float64)
    o = np.empty((len(rows), Hq, hd), np.float64)
    for i, t in enumerate(rows):
        for h in range(Hq):
            s = kf[:t + 1, h // G] @ qf[i, h] * (1.0 / math.sqrt(hd))
            s = np.exp(s - s.max())
            o[i, h] = (s / s.sum()) @ vf[:t + 1, h // G]
    o2 = oracle.f32_to_bf16(o.astype(np.float32)).reshape(len(rows), nq)
    xr = np.ascontiguousarray(xs[rows])
    x2 = _op(oracle, "Add", [xr, _op(oracle, "MatMul", [o2, x["w_o"]])])
    h2 = _op(oracle, "RMSNorm", [x2, x["w_ln2"]], eps=eps)
    gt = _op(oracle, "MatMul", [h2, x["w_gate"]])
    up = _op(oracle, "MatMul", [h2, x["w_up"]])
    mm = _op(oracle, "Mul", [_op(oracle, "SiLU", [gt]), up])
    return _op(oracle, "Add", [x2, _op(oracle, "MatMul", [mm, x["w_down"]])])


def test_c5_prefill_b8_s4096_full_size(vtc, oracle):
    from paper_2604_09558_b200 import workloads as W
    B, S = 8, 4096
    doc = W.llama_prefill_layer(B=B, S=S)
    rng = np.random.default_rng(51)
    cos, sin = W.rope_tables_prefill(B, S)
    x = _inputs(doc, rng, W.llama_weight_scales(),
                {"cos": oracle.f32_to_bf16(cos.astype(np.float32)), "sin": oracle.f32_to_bf16(sin.astype(np.float32))})
    g = vtc.parse_graph(doc)
    p = vtc.Plan(g, vtc.MAX_ELIMINATION)
    kinds = _kernels(p)
    assert p.info()["data_movement_launches"] == 0
    assert kinds.count("gemm_tc_bf16") >= 4 and "attn_fmha_tc" in kinds, kinds
    got = vtc.execute(g, p, x)["y"]
    rows = [0, 1, 2047, 4095]
    errs = []
    for seq in (0, 7):
        want = _prefill_rows_oracle(oracle, x, seq, rows, S)
        errs.append(_relerr(oracle.bf16_to_f32(got[[seq * S + t for t in rows]]), oracle.bf16_to_f32(want)))
    print(f"C5 full size: max rel err per sequence {errs}")
    assert max(errs) < 2e-2, errs

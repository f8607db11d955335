"""tcgen05 / TMEM flash attention (csrc/k_attn_fmha.cu) against the fp64
restatement (oracle/vtc_oracle.py Attention) at the north-star bf16 tolerance
(||err||_inf / ||ref||_inf < 2e-2), through virtual Q / K / V / O maps: the
[B,S,H,d] -> [B,H,S,d] transposes and the GQA Unsqueeze / Expand / Reshape are
views the host proves affine and hands to TMA.  Edge cases: ragged S (partial
query and key tiles), Sq < Sk (causal offset), non-causal, GQA 1 / 2 / 4, the
mma.sync kernel (VTC_NO_FMHA) as a second implementation."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def attn_graph(B, Sq, Sk, H, Hkv, causal, hd=128):
    from paper_2604_09558_b200.workloads import GraphBuilder
    G = H // Hkv
    g = GraphBuilder("bf16")
    g.input("q", [B, Sq, H, hd])
    g.input("k", [B, Sk, Hkv, hd])
    g.input("v", [B, Sk, Hkv, hd])
    g.node("q_t", "Transpose", ["q"], "qh", {"perm": [0, 2, 1, 3]})
    for t in ("k", "v"):
        g.node(f"{t}_t", "Transpose", [t], f"{t}t", {"perm": [0, 2, 1, 3]})          # [B, Hkv, Sk, d]
        g.node(f"{t}_u", "Unsqueeze", [f"{t}t"], f"{t}u", {"axis": 2})                # [B, Hkv, 1, Sk, d]
        g.node(f"{t}_e", "Expand", [f"{t}u"], f"{t}e", {"shape": [B, Hkv, G, Sk, hd]})
        g.node(f"{t}_r", "Reshape", [f"{t}e"], f"{t}h", {"shape": [B, H, Sk, hd]})
    g.node("attn", "Attention", ["qh", "kh", "vh"], "oh", {"scale": 1.0 / np.sqrt(hd), "causal": causal})
    g.node("o_t", "Transpose", ["oh"], "o", {"perm": [0, 2, 1, 3]}, out_kind="output")  # [B, Sq, H, d]
    return g.doc()


CASES = [
    dict(B=1, Sq=128, Sk=128, H=2, Hkv=1, causal=True),
    dict(B=2, Sq=300, Sk=300, H=4, Hkv=2, causal=True),     # ragged: partial query and key tiles
    dict(B=1, Sq=512, Sk=512, H=2, Hkv=2, causal=False),
    dict(B=1, Sq=128, Sk=384, H=4, Hkv=1, causal=True),     # chunked prefill: keys [0, q + 256]
    dict(B=2, Sq=1024, Sk=1024, H=8, Hkv=2, causal=True),
]


@pytest.mark.parametrize("cfg", CASES)
def test_fmha_matches_fp64_reference(vtc, oracle, cfg):
    doc = attn_graph(**cfg)
    x = oracle.random_inputs(doc, seed=3)
    want = oracle.bf16_to_f32(oracle.execute(doc, x)["o"]).astype(np.float64)
    g = vtc.parse_graph(doc)
    p = vtc.Plan(g, vtc.MAX_ELIMINATION)
    kinds = [l["kernel"] for l in p.info(dry=True)["launches"]]
    assert kinds == ["attn_fmha_tc"], kinds
    got = vtc.bf16_to_f32(vtc.execute(g, p, x)["o"]).astype(np.float64)
    err = float(np.max(np.abs(got - want)) / np.max(np.abs(want)))
    print(cfg, "rel err", err)
    assert err < 2e-2, err


def test_fmha_equals_mma_sync_kernel_within_tolerance(vtc, oracle):
    """The same layer through the round-1 mma.sync flash kernel (VTC_NO_FMHA=1,
    a separate process: the switch is read at plan time)."""
    cfg = dict(B=2, Sq=256, Sk=256, H=4, Hkv=2, causal=True)
    doc = attn_graph(**cfg)
    x = oracle.random_inputs(doc, seed=5)
    g = vtc.parse_graph(doc)
    a = vtc.bf16_to_f32(vtc.execute(g, vtc.Plan(g, vtc.MAX_ELIMINATION), x)["o"])
    os.environ["VTC_NO_FMHA"] = "1"
    try:
        p2 = vtc.Plan(g, vtc.MAX_ELIMINATION)
        assert [l["kernel"] for l in p2.info(dry=True)["launches"]] == ["attn_prefill_tc"]
        b = vtc.bf16_to_f32(vtc.execute(g, p2, x)["o"])
    finally:
        del os.environ["VTC_NO_FMHA"]
    assert float(np.max(np.abs(a - b)) / np.max(np.abs(b))) < 2e-2


WINDOW_CASES = [
    dict(B=3, Sq=49, Sk=49, H=3, Hkv=3, causal=False, hd=32),   # a Swin window
    dict(B=2, Sq=64, Sk=64, H=4, Hkv=2, causal=True, hd=64),    # full tile, GQA, causal
    dict(B=5, Sq=17, Sk=40, H=2, Hkv=1, causal=True, hd=32),    # ragged, causal offset Sk - Sq
]


@pytest.mark.parametrize("cfg", WINDOW_CASES)
def test_window_attention_matches_fp64_reference(vtc, oracle, cfg):
    """Short-sequence attention (one warp per (batch, head) item, all keys in one
    64-key tile, single-pass softmax) through the transposed / GQA-expanded views."""
    doc = attn_graph(**cfg)
    x = oracle.random_inputs(doc, seed=9)
    want = oracle.bf16_to_f32(oracle.execute(doc, x)["o"]).astype(np.float64)
    g = vtc.parse_graph(doc)
    p = vtc.Plan(g, vtc.MAX_ELIMINATION)
    assert [l["kernel"] for l in p.info(dry=True)["launches"]] == ["attn_window_tc"]
    got = vtc.bf16_to_f32(vtc.execute(g, p, x)["o"]).astype(np.float64)
    err = float(np.max(np.abs(got - want)) / np.max(np.abs(want)))
    assert err < 2e-2, err

"""GPU regression tests for executor invariants (round-1 review findings):

* rebinding a root between two vtc_run calls must not replay a graph that
  still holds the old (freed) address;
* an input staged by an earlier vtc_run call and not named in a later one keeps
  its contents when the staging arena is rebuilt;
* a horizontally fused tcgen05 launch with a narrow first matrix at prefill M
  (K split forced) stays correct;
* a sibling MatMul is only absorbed into an earlier launch when everything it
  reads is produced before that launch.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _relerr(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want)) / max(1e-30, float(np.max(np.abs(want)))))


def _small_layer(oracle, W, seed=5):
    cfg = dict(B=2, L=64, pos=40, D=256, Hq=4, Hkv=2, hd=64, F=512)
    doc = W.llama_decode_layer(**cfg)
    x = oracle.random_inputs(doc, seed=seed, scales=W.llama_weight_scales(cfg["D"], cfg["F"]))
    cos, sin = W.rope_tables(cfg["B"], [cfg["pos"]] * cfg["B"], hd=cfg["hd"])
    x["cos"] = oracle.f32_to_bf16(cos.astype(np.float32))
    x["sin"] = oracle.f32_to_bf16(sin.astype(np.float32))
    return cfg, doc, x


def test_rebind_root_between_runs_uses_the_new_buffer(vtc, oracle):
    from paper_2604_09558_b200 import workloads as W
    cfg, doc, x = _small_layer(oracle, W)
    g = vtc.parse_graph(doc)
    p = vtc.Plan(g, vtc.MAX_ELIMINATION)
    for k, v in x.items():
        p.upload(k, v)
    first = p.run({"x": x["x"]}, ["y"])["y"]
    # a second plan holds different O-projection weights; p's w_o root is rebound to them
    w_o2 = oracle.f32_to_bf16(np.random.default_rng(9).uniform(-1, 1, x["w_o"].shape).astype(np.float32) / 16)
    q = vtc.Plan(g, vtc.MAX_ELIMINATION)
    q.upload("w_o", w_o2)
    p.bind_root("w_o", q.root_ptr("w_o"))
    second = p.run({"x": x["x"]}, ["y"])["y"]
    want = oracle.execute(doc, dict(x, w_o=w_o2))["y"]
    assert not np.array_equal(first, second)
    assert _relerr(oracle.bf16_to_f32(second), oracle.bf16_to_f32(want)) < 2e-2
    fresh = vtc.execute(g, vtc.Plan(g, vtc.MAX_ELIMINATION), dict(x, w_o=w_o2))["y"]
    assert np.array_equal(second, fresh)


def test_staged_inputs_survive_an_arena_rebuild(vtc, oracle):
    from paper_2604_09558_b200 import workloads as W
    cfg, doc, x = _small_layer(oracle, W)
    g = vtc.parse_graph(doc)
    p = vtc.Plan(g, vtc.MAX_ELIMINATION)
    for k, v in x.items():
        p.upload(k, v)
    # call 1 stages x, the norm weights and the RoPE tables; call 2 names only x
    small = {k: x[k] for k in ("x", "w_ln1", "w_ln2", "cos", "sin")}
    p.run(small, ["y"])
    xs = oracle.f32_to_bf16(np.random.default_rng(4).uniform(-1, 1, x["x"].shape).astype(np.float32))
    got = p.run({"x": xs}, ["y"])["y"]
    want = vtc.execute(g, vtc.Plan(g, vtc.MAX_ELIMINATION), dict(x, x=xs))["y"]
    assert np.array_equal(got, want)


def test_fused_siblings_with_narrow_first_matrix_at_prefill_m(vtc, oracle):
    from paper_2604_09558_b200.workloads import GraphBuilder
    M, K, N1, N2 = 4096, 512, 1024, 4096
    g = GraphBuilder("bf16")
    g.input("a", [M, K])
    g.input("w1", [K, N1])
    g.input("w2", [K, N2])
    g.node("mm1", "MatMul", ["a", "w1"], "y1", out_kind="output")
    g.node("mm2", "MatMul", ["a", "w2"], "y2", out_kind="output")
    doc = g.doc()
    x = oracle.random_inputs(doc, seed=12, scales={"w1": 1 / np.sqrt(K), "w2": 1 / np.sqrt(K)})
    gr = vtc.parse_graph(doc)
    p = vtc.Plan(gr, vtc.MAX_ELIMINATION)
    assert any(l["node"] == "mm1+mm2" for l in p.info(dry=True)["launches"])
    got = vtc.execute(gr, p, x)
    a = oracle.bf16_to_f32(x["a"]).astype(np.float64)
    for y, w in (("y1", "w1"), ("y2", "w2")):
        want = a @ oracle.bf16_to_f32(x[w]).astype(np.float64)
        assert _relerr(oracle.bf16_to_f32(got[y]), want) < 1e-2, y


@pytest.mark.parametrize("M", [2, 64])
def test_sibling_reading_a_late_weight_is_not_hoisted(vtc, oracle, M):
    """mm_a's weight is computed (w = wa + wb) and so runs late in topological
    order; mm_b (same A, graph-input weight) listed after it must not be absorbed
    into mm_a's launch ahead of mm_b's own consumer."""
    from paper_2604_09558_b200.workloads import GraphBuilder
    K, N = 256, 512
    g = GraphBuilder("bf16")
    g.input("h", [M, K])
    g.input("wa", [K, N])
    g.input("wb", [K, N])
    g.input("w2", [K, N])
    g.input("r", [M, N])
    g.node("mm_a", "MatMul", ["h", "w"], "ya")
    g.node("mm_b", "MatMul", ["h", "w2"], "yb")
    g.node("use_b", "Add", ["yb", "r"], "zb", out_kind="output")
    g.node("mk_w", "Add", ["wa", "wb"], "w")
    g.node("out", "Add", ["ya", "zb"], "y", out_kind="output")
    doc = g.doc()
    sc = 1 / np.sqrt(2 * K)
    x = oracle.random_inputs(doc, seed=M, scales={"wa": sc, "wb": sc, "w2": sc})
    want = oracle.execute(doc, x)
    gr = vtc.parse_graph(doc)
    got = vtc.execute(gr, vtc.Plan(gr, vtc.MAX_ELIMINATION), x)
    for k in ("y", "zb"):
        assert _relerr(oracle.bf16_to_f32(got[k]), oracle.bf16_to_f32(want[k])) < 2e-2, k

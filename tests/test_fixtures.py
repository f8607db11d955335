"""Paper case-study fixtures (SPEC.md acceptance 7).

YOLOv11 C3K2 block: y0 = x.W_cv1 -> Split(a, b) -> bottleneck e = b + SiLU(b.W_m1).W_m2
-> Y = Concat(a, b, e) -> Y.W_cv2.  Its two data-movement operators (Split and
Concat) run as copy kernels in the all-physical plan and vanish under VTC:
the paper's strategy makes a, b, e (and the cv1 output y0) virtual tensors of
Y, so cv1 and the bottleneck's residual Add store straight into Y's channel
ranges.  Host-side checks here (plans are built dry); GPU parity in
tests/test_gpu.py::test_c3k2_block_strategies_bit_identical.
"""
import pytest

C3K2 = dict(N=4096, c=64, cin=128, cout=128)


def paper_strategy(g):
    """VTOG edges of the Fig. 11 strategy: a, b, e over Y (Concat eliminated
    by its inputs) and y0 over a / b (Split eliminated by its input)."""
    want = {("a", "Y"), ("b", "Y"), ("e", "Y"), ("y0", "a"), ("y0", "b")}
    return [e["id"] for e in g.vtog()["edges"] if (e["src"], e["dst"]) in want]


def dm_ops(info):
    return {l["node"] for l in info["launches"] if l["kernel"] == "gather_copy"}


def test_c3k2_materialised_plan_runs_split_and_concat(vtc):
    from paper_2604_09558_b200 import workloads as W
    g = vtc.parse_graph(W.c3k2_block(**C3K2))
    info = vtc.Plan(g, vtc.MATERIALIZE).info(dry=True)
    assert dm_ops(info) == {"split", "concat"}


def test_c3k2_paper_strategy_makes_a_b_e_virtual_over_Y(vtc):
    from paper_2604_09558_b200 import workloads as W
    g = vtc.parse_graph(W.c3k2_block(**C3K2))
    sel = paper_strategy(g)
    assert len(sel) == 5
    p = vtc.Plan(g, vtc.SELECTED, sel)
    info = p.info(dry=True)
    assert info["data_movement_launches"] == 0 and not dm_ops(info)
    assert sorted(info["eliminated_ops"]) == ["concat", "split"]
    assert "Y" in info["roots"]
    for t in ("a", "b", "e", "y0"):
        assert t not in info["roots"]
        assert p.map_json(t)["targets"] == ["Y"], t
    # the two stores land in disjoint channel ranges of Y (row pitch 3c)
    assert "Y@128+192*i0" in p.map_json("e")["text"]
    # no gather GEMM: cv2 reads a plain Y
    kinds = {l["node"]: l["kernel"] for l in info["launches"]}
    assert kinds["cv2"] == "gemm_tc_bf16"


def test_c3k2_max_elimination_also_eliminates_both(vtc):
    from paper_2604_09558_b200 import workloads as W
    g = vtc.parse_graph(W.c3k2_block(**C3K2))
    info = vtc.Plan(g, vtc.MAX_ELIMINATION).info(dry=True)
    assert info["data_movement_launches"] == 0
    assert sorted(info["eliminated_ops"]) == ["concat", "split"]

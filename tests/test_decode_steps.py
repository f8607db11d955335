"""Multi-step decode with a runtime position.

One plan (FLAG_DYNAMIC_POS, built with the graph's ScatterND row = L - 1) and
one captured graph serve consecutive decode steps: each step writes the new
token's K / V at `pos` and attends over keys [0, pos], with `pos` read on the
device (the vtc_run input "__pos" or Plan.set_position).  The oracle replays
the same steps with the reference's static-index graph (ScatterND [[pos]],
Slice [0, pos + 1)) on its own evolving cache.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _relerr(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want)) / max(1e-30, float(np.max(np.abs(want)))))


@pytest.mark.parametrize("cfg", [
    dict(B=2, L=64, D=256, Hq=4, Hkv=2, hd=64, F=512),      # streamed GEMV path (M <= 4), fused RoPE epilogue
    dict(B=32, L=96, D=256, Hq=4, Hkv=2, hd=128, F=512),    # tcgen05 GEMM, RoPE trees in its epilogue
    dict(B=64, L=256, D=4096, Hq=32, Hkv=8, hd=128, F=14336),  # C3 widths: split-K GEMMs, trees spread over splits
    dict(B=1, L=2048, D=4096, Hq=32, Hkv=8, hd=128, F=14336),  # BASELINE configs[1] shape
])
def test_dynamic_position_consecutive_steps(vtc, oracle, cfg):
    _consecutive_steps(vtc, oracle, cfg)


def test_dynamic_position_rope_trees_in_split_k_epilogue(vtc, oracle, monkeypatch):
    # opt-in (VTC_TREE_COOP=1): the Q / K RoPE trees run in the cooperative split-K epilogue of
    # the decode QKV GEMM, the roped K row stored into the cache at the runtime position
    monkeypatch.setenv("VTC_TREE_COOP", "1")
    launches = _consecutive_steps(vtc, oracle, dict(B=64, L=256, D=4096, Hq=32, Hkv=8, hd=128, F=14336))
    assert "eltwise_aff" not in launches and "eltwise" not in launches, launches


def _consecutive_steps(vtc, oracle, cfg):
    from paper_2604_09558_b200 import workloads as W
    B, L, hd = cfg["B"], cfg["L"], cfg["hd"]
    doc = W.llama_decode_layer(**cfg)  # ScatterND row L - 1: the largest position
    x0 = oracle.random_inputs(doc, seed=17, scales=W.llama_weight_scales(cfg["D"], cfg["F"]))
    g = vtc.parse_graph(doc)
    p = vtc.Plan(g, vtc.MAX_ELIMINATION, flags=vtc.FLAG_DYNAMIC_POS)
    for k, v in x0.items():
        p.upload(k, v)
    launches = [l["kernel"] for l in p.info(dry=True)["launches"]]
    assert p.info(dry=True)["data_movement_launches"] == 0
    kc, vc = x0["k_cache"].copy(), x0["v_cache"].copy()
    rng = np.random.default_rng(5)
    start = L - 10
    errs = []
    for step in range(8):
        pos = start + step
        xs = oracle.f32_to_bf16(rng.uniform(-1, 1, size=(B, cfg["D"])).astype(np.float32))
        cos, sin = W.rope_tables(B, [pos] * B, hd=hd)
        cos, sin = oracle.f32_to_bf16(cos.astype(np.float32)), oracle.f32_to_bf16(sin.astype(np.float32))
        ref_doc = W.llama_decode_layer(**cfg, pos=pos)
        env = oracle.execute(ref_doc, dict(x0, x=xs, cos=cos, sin=sin, k_cache=kc, v_cache=vc), keep_all=True)
        kc, vc = env["kc2"], env["vc2"]
        if step % 2 == 0:  # the position as a vtc_run input
            got = p.run({"x": xs, "cos": cos, "sin": sin, "__pos": np.array([pos], np.int64)}, ["y"])["y"]
        else:  # or set on the plan, then upload / execute / download
            p.set_position(pos)
            for k, v in (("x", xs), ("cos", cos), ("sin", sin)):
                p.upload(k, v)
            p.execute_graph()
            got = p.download("y")
        errs.append(_relerr(oracle.bf16_to_f32(got), oracle.bf16_to_f32(env["y"])))
    print(f"dynamic position {cfg}: rel err per step {np.round(errs, 5).tolist()}")
    assert max(errs) < 2e-2, errs
    assert [l["kernel"] for l in p.info()["launches"]] == launches
    # the cache rows of the 8 positions hold the steps' K / V; every other row is untouched
    gk, gv = p.download("k_cache"), p.download("v_cache")
    rows = slice(start, start + 8)
    assert _relerr(oracle.bf16_to_f32(gk[rows]), oracle.bf16_to_f32(kc[rows])) < 2e-2
    assert _relerr(oracle.bf16_to_f32(gv[rows]), oracle.bf16_to_f32(vc[rows])) < 2e-2
    keep = np.r_[0:start, start + 8:L]
    assert np.array_equal(gk[keep], x0["k_cache"][keep]) and np.array_equal(gv[keep], x0["v_cache"][keep])
    return launches


def test_dynamic_position_errors(vtc, oracle):
    from paper_2604_09558_b200 import workloads as W
    doc = W.llama_decode_layer(B=2, L=64, D=256, Hq=4, Hkv=2, hd=64, F=512)
    g = vtc.parse_graph(doc)
    p = vtc.Plan(g, vtc.MAX_ELIMINATION, flags=vtc.FLAG_DYNAMIC_POS)
    with pytest.raises(vtc.api.ERRORS[6]):  # OutOfBoundsError
        p.set_position(64)
    # an all-physical plan clones the cache (no in-place update): no dynamic position
    with pytest.raises(vtc.api.ERRORS[22]):  # UnsupportedError
        vtc.Plan(g, vtc.MATERIALIZE, flags=vtc.FLAG_DYNAMIC_POS).prepare()
    # the strong comparator (ScatterND in place, every other copy materialised) supports it
    pm = vtc.Plan(g, vtc.INPLACE_UPDATES, flags=vtc.FLAG_DYNAMIC_POS)
    pm.prepare()
    with pytest.raises(vtc.api.ERRORS[16]):  # ExecutionError: static plan
        vtc.Plan(g, vtc.MAX_ELIMINATION).set_position(3)


def test_inplace_updates_comparator_matches_and_copies_only_the_slab(vtc, oracle):
    """The strong materialising comparator: ScatterND writes its slab in place,
    every other data-movement op is a copy kernel; same result as the VTC plan."""
    from paper_2604_09558_b200 import workloads as W
    cfg = dict(B=2, L=64, pos=40, D=256, Hq=4, Hkv=2, hd=64, F=512)
    doc = W.llama_decode_layer(**cfg)
    x = oracle.random_inputs(doc, seed=5, scales=W.llama_weight_scales(cfg["D"], cfg["F"]))
    cos, sin = W.rope_tables(2, [40, 40], hd=64)
    x["cos"], x["sin"] = oracle.f32_to_bf16(cos.astype(np.float32)), oracle.f32_to_bf16(sin.astype(np.float32))
    g = vtc.parse_graph(doc)
    pv, pi = vtc.Plan(g, vtc.MAX_ELIMINATION), vtc.Plan(g, vtc.INPLACE_UPDATES)
    yv = vtc.execute(g, pv, x, roots=("k_cache",))
    yi = vtc.execute(g, pi, x, roots=("k_cache",))
    info = pi.info()
    assert info["data_movement_launches"] > 10
    scat = [l for l in info["launches"] if l["node"] in ("k_scatter", "v_scatter")]
    assert len(scat) == 2 and all(l["bytes"] <= 4 * 2 * 2 * 64 for l in scat), scat  # one row, not the cache
    want = oracle.execute(doc, x)["y"]
    assert _relerr(oracle.bf16_to_f32(yi["y"]), oracle.bf16_to_f32(want)) < 2e-2
    assert _relerr(oracle.bf16_to_f32(yi["y"]), oracle.bf16_to_f32(yv["y"])) < 2e-2
    assert np.array_equal(np.delete(yi["root:k_cache"], 40, 0), np.delete(x["k_cache"], 40, 0))

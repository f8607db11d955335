"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED
reference library (oracle/_ref/libvtelim_ref.so, built by oracle/Makefile from
/root/reference/proj/src).  Run here, where /root/reference exists:

    make -C oracle && python tests/golden/make_golden.py

Writes
  * ref_small.npz  -- per case: the reference's seeded inputs
    (make_random_inputs, proj/src/executor.cpp:508-528) and its execute()
    outputs (all-physical plan, proj/src/executor.cpp:500-506) for small
    graphs of every data-movement operator, the C1 chain and the frame-2 chain;
  * ref_digests.json -- FNV-1a-64 digests (proj/src/executor.cpp:86-94) of the
    reference outputs for cases too large to store (C1 at full size).
The fixtures pin the numpy oracle (tests/test_golden.py, CPU) and the CUDA
path (tests/test_gpu.py, B200) to the reference itself.
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import ref  # noqa: E402
from paper_2604_09558_b200 import workloads as W  # noqa: E402
from paper_2604_09558_b200.workloads import GraphBuilder  # noqa: E402


def fnv1a64(a: np.ndarray) -> int:
    """array_digest (proj/src/executor.cpp:86-94): FNV-1a-64 over the raw bytes."""
    h = 1469598103934665603
    for b in np.ascontiguousarray(a).view(np.uint8).tobytes():
        h = ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def cases():
    out = {}
    for dt in ("f64", "f32", "i64"):
        for kind, shape, attrs in [
            ("Transpose", [3, 4, 5], {"perm": [2, 0, 1]}),
            ("Reshape", [3, 4, 5], {"shape": [6, 10]}),
            ("Unsqueeze", [3, 4, 5], {"axis": 1}),
            ("Slice", [6, 4, 5], {"axes": [0, 2], "starts": [1, 2], "ends": [5, 5]}),
            ("Expand", [2, 3, 4], {"shape": [2, 9, 4]}),
            ("Expand", [2, 1, 4], {"shape": [2, 5, 4]}),
        ]:
            g = GraphBuilder(dt)
            g.input("x", shape)
            g.node("op", kind, ["x"], "y", attrs, out_kind="output")
            out[f"{kind.lower()}_{len(out)}_{dt}"] = g.doc()
        g = GraphBuilder(dt)
        g.input("x", [4, 6])
        g.input("z", [4, 2])
        g.node("s", "Split", ["x"], ["a", "b"], {"axis": 1, "sizes": [2, 4]}, out_kind="output")
        g.node("c", "Concat", ["z", "b"], "y", {"axis": 1}, out_kind="output")
        g.input("d", [5, 3, 2])
        g.input("u", [2, 3, 2])
        g.node("sc", "ScatterND", ["d", "u"], "w", {"indices": [[4], [1]]}, out_kind="output")
        out[f"split_concat_scatter_{dt}"] = g.doc()
    out["c1_chain_64_f32"] = W.c1_chain(64)
    out["frame2_b1_l18_f32"] = W.frame2_subgraph(B=1, L=18)
    out["frame2_b2_l24_f64"] = W.frame2_subgraph(B=2, L=24, dtype="f64")
    return out


def main():
    assert ref.available(), "build oracle/_ref first (make -C oracle)"
    arrays, index = {}, {}
    for name, doc in cases().items():
        rg = ref.RefGraph(doc)
        x = rg.inputs_random(5)
        y, _, _ = rg.plan().execute(x)
        index[name] = {"doc": doc, "inputs": sorted(x), "outputs": sorted(y)}
        for k, v in x.items():
            arrays[f"{name}/in/{k}"] = v
        for k, v in y.items():
            arrays[f"{name}/out/{k}"] = v
    np.savez_compressed(HERE / "ref_small.npz", **arrays)
    (HERE / "ref_small.json").write_text(json.dumps(index, indent=0, sort_keys=True))
    # C1 at full size: the reference's own seeded inputs and output digest
    rg = ref.RefGraph(W.c1_chain(1024))
    x = rg.inputs_random(1)
    plan = rg.plan()
    y, ns, _ = plan.execute(x)
    dig = {"c1_chain_1024_f32_seed1": {"y": format(fnv1a64(y["y"]), "016x"), "reference_execute_ms": ns / 1e6}}
    (HERE / "ref_digests.json").write_text(json.dumps(dig, indent=1))
    print(f"{len(index)} small cases, digests {dig}")


if __name__ == "__main__":
    main()

"""Run one tcgen05 GEMM shape (argv M K N) and compare with float64."""
import sys
import numpy as np
sys.path.insert(0, "oracle")
sys.path.insert(0, ".")
import vtc_oracle as O
import paper_2604_09558_b200 as vtc
from paper_2604_09558_b200.workloads import GraphBuilder
M, K, N = map(int, sys.argv[1:4])
g = GraphBuilder("bf16")
g.input("a", [M, K]); g.input("w", [K, N])
g.node("mm", "MatMul", ["a", "w"], "y", out_kind="output")
doc = g.doc()
x = O.random_inputs(doc, seed=3, scales={"w": 1.0 / np.sqrt(K)})
G = vtc.parse_graph(doc)
p = vtc.Plan(G, vtc.MAX_ELIMINATION)
print([l["kernel"] for l in p.info(dry=True)["launches"]], flush=True)
got = vtc.execute(G, p, x)["y"]
want = O.bf16_to_f32(x["a"]).astype(np.float64) @ O.bf16_to_f32(x["w"]).astype(np.float64)
err = np.max(np.abs(O.bf16_to_f32(got) - want)) / np.max(np.abs(want))
print(M, K, N, "relerr", err, flush=True)

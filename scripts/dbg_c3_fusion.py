import os
os.environ["VTC_DEBUG_FUSION"] = "1"
from paper_2604_09558_b200 import api as vtc, workloads as W
doc = W.llama_decode_layer(B=64, L=8192)
g = vtc.parse_graph(doc)
p = vtc.Plan(g, vtc.MAX_ELIMINATION, flags=vtc.FLAG_DYNAMIC_POS)
print("dry", [l["node"][:50] for l in p.info(dry=True)["launches"]], flush=True)
p.prepare()
print("real", [l["node"][:50] for l in p.info()["launches"]], flush=True)

import os, sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
os.environ["VTC_TRACE"] = "1"
import bench, paper_2604_09558_b200 as vtc
from paper_2604_09558_b200 import workloads as W
cfg = bench.CONFIGS["c2"]; dev = torch.device("cuda", 0); stream = torch.cuda.current_stream()
doc = W.llama_decode_layer(B=1, L=2048); g = vtc.parse_graph(doc)
dt, host = bench.build_layer_inputs(doc, cfg, torch, dev)
p = vtc.Plan(g, vtc.MAX_ELIMINATION)
for k, t in dt.items(): p.bind_root(k, t.data_ptr())
for k, t in host.items(): p.upload_ptr(k, t.data_ptr(), t.numel() * t.element_size(), stream)
p.prepare()
for _ in range(5): p.execute_graph(stream)
torch.cuda.synchronize(); p.trace()
for _ in range(1): p.execute_graph(stream)
torch.cuda.synchronize(); tr = p.trace()
print("qkv row:", [int(x) for x in tr[0]])

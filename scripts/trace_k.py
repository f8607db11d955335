"""Per-launch device trace of one config's VTC plan (VTC_TRACE=1): entry / exit
(ns, relative to the first entry) and the kernel accumulators 2..7 (sums over
CTAs: gemm_tc 2 = mainloop, 3 = epilogue, 4 = CTA count).  python scripts/trace_k.py c3"""
import os
import sys

sys.path.insert(0, "."); sys.path.insert(0, "oracle")
os.environ["VTC_TRACE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_09558_b200 as vtc  # noqa: E402
from paper_2604_09558_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = bench.CONFIGS[name]
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream().cuda_stream
if cfg.get("swin"):
    doc = W.swin_block(B=cfg["B"], H=cfg["H"])
elif cfg.get("prefill"):
    doc = W.llama_prefill_layer(B=cfg["B"], S=cfg["S"])
else:
    doc = W.llama_decode_layer(B=cfg["B"], L=cfg["L"])
g = vtc.parse_graph(doc)
dt, host = bench.build_layer_inputs(doc, cfg, torch, dev)
p = vtc.Plan(g, vtc.MAX_ELIMINATION)
for k, t in dt.items():
    p.bind_root(k, t.data_ptr())
for k, t in host.items():
    p.upload_ptr(k, t.data_ptr(), t.numel() * t.element_size(), stream)
p.prepare()
for _ in range(5):
    p.execute_graph(stream)
torch.cuda.synchronize()
p.trace()
p.execute_graph(stream)
torch.cuda.synchronize()
tr = p.trace().astype(np.int64)
t0 = tr[:, 0][tr[:, 0] > 0].min()
for l, row in zip(p.info()["launches"], tr):
    print(f"{l['node'][:40]:40s} {l['kernel']:24s} entry {(row[0]-t0)/1e3:8.2f} exit {(row[1]-t0)/1e3:8.2f} us  acc",
          [round((int(x) - t0) / 1e3, 2) if x > 10**17 else int(x) for x in row[2:8]])

"""Run one configuration's VTC plan a few times (for ncu captures of single kernels):
python scripts/run_plan.py c4 [reps]"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2604_09558_b200 as vtc  # noqa: E402
from paper_2604_09558_b200 import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = bench.CONFIGS[name]
if cfg.get("swin"):
    doc = W.swin_block(B=cfg["B"], H=cfg["H"])
elif cfg.get("prefill"):
    doc = W.llama_prefill_layer(B=cfg["B"], S=cfg["S"])
else:
    doc = W.llama_decode_layer(B=cfg["B"], L=cfg["L"])
dev = torch.device("cuda:0")
stream = torch.cuda.current_stream().cuda_stream
g = vtc.parse_graph(doc)
dev_tensors, host = bench.build_layer_inputs(doc, cfg, torch, dev)
p = vtc.Plan(g, vtc.MAX_ELIMINATION)
for tid, t in dev_tensors.items():
    p.bind_root(tid, t.data_ptr())
for tid, t in host.items():
    p.upload_ptr(tid, t.data_ptr(), t.numel() * t.element_size(), stream)
p.prepare()
print([l["node"] + ":" + l["kernel"] for l in p.info()["launches"]], flush=True)
for _ in range(reps):
    p.execute_graph(stream) if os.environ.get("GRAPH", "0") == "1" else p.execute(stream)
torch.cuda.synchronize()
print("done")

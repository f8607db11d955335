"""One C5 layer plan (B=8, S=4096), prepared and executed once (eager) -- for ncu captures."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import paper_2604_09558_b200 as vtc  # noqa: E402
from paper_2604_09558_b200 import workloads as W  # noqa: E402
g = vtc.parse_graph(W.llama_prefill_layer(B=8, S=4096))
p = vtc.Plan(g, vtc.MAX_ELIMINATION)
p.prepare()
s = torch.cuda.Stream()
for _ in range(2):
    p.execute(s.cuda_stream)
torch.cuda.synchronize()
print([l["kernel"] for l in p.info()["launches"]])

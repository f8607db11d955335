"""C2 (decode B=1, KV 2048) device timeline: per launch first-CTA entry / last-CTA
exit relative to the step start and the kernel checkpoints, averaged over replays."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
os.environ["VTC_TRACE"] = "1"
import torch  # noqa: E402

import paper_2604_09558_b200 as vtc  # noqa: E402
from paper_2604_09558_b200 import workloads as W  # noqa: E402

B = int(os.environ.get("C2_B", "1"))
L = int(os.environ.get("C2_L", "2048"))
doc = W.llama_decode_layer(B=B, L=L, pos=L - 1)
g = vtc.parse_graph(doc)
p = vtc.Plan(g, vtc.MAX_ELIMINATION)
p.prepare()
rng = np.random.default_rng(0)
for t, spec in g.tensors().items():
    if spec["kind"] == "input":
        n = int(np.prod(spec["shape"]))
        p.upload(t, vtc.f32_to_bf16((rng.uniform(-1, 1, n) * 0.02).astype(np.float32)).reshape(spec["shape"]))
s = torch.cuda.Stream()
for _ in range(5):
    p.execute_graph(s.cuda_stream)
torch.cuda.synchronize()
launches = p.info()["launches"]
acc = None
R = 20
for _ in range(R):
    p.trace()
    p.execute_graph(s.cuda_stream)
    torch.cuda.synchronize()
    tr = p.trace().astype(np.float64)
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    rel = tr.copy()
    rel[:, :2] -= t0
    # checkpoints recorded as absolute globaltimer values (trace_point) -> relative too
    big = rel[:, 2:] > 1e15
    rel[:, 2:][big] -= t0
    acc = rel if acc is None else acc + rel
acc /= R
for l, row in zip(launches, acc):
    print(f"{l['kernel']:28s} {l['node'][:40]:40s} entry {row[0]/1e3:7.2f} us  exit {row[1]/1e3:7.2f} us  dur {(row[1]-row[0])/1e3:6.2f}  "
          f"bytes {l['bytes']/1e6:7.2f} MB  ck {[round(x/1e3, 2) for x in row[2:]]}")

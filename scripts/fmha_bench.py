"""C5's attention alone (B=8, S=4096, 32 query / 8 KV heads, d=128, causal) through
the attention-only graph of tests/test_gpu_fmha.py: device time per launch
(CUDA-graph replay, CUDA events) and TFLOP/s against the measured bf16 peak.
--once: a single execution (for ncu)."""
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402

import paper_2604_09558_b200 as vtc  # noqa: E402
from test_gpu_fmha import attn_graph  # noqa: E402

B, S, H, HKV = (int(x) for x in os.environ.get("FMHA_SHAPE", "8,4096,32,8").split(","))
causal = os.environ.get("FMHA_CAUSAL", "1") == "1"
doc = attn_graph(B=B, Sq=S, Sk=S, H=H, Hkv=HKV, causal=causal)
g = vtc.parse_graph(doc)
p = vtc.Plan(g, vtc.MAX_ELIMINATION)
p.prepare()
rng = np.random.default_rng(0)
for t in ("q", "k", "v"):
    shp = g.tensors()[t]["shape"]
    p.upload(t, vtc.f32_to_bf16(rng.uniform(-1, 1, size=shp).astype(np.float32)))
s = torch.cuda.Stream()
if "--once" in sys.argv:
    p.execute(s.cuda_stream)
    torch.cuda.synchronize()
    sys.exit(0)
for _ in range(3):
    p.execute_graph(s.cuda_stream)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(10):
    a.record(s)
    p.execute_graph(s.cuda_stream)
    b.record(s)
    b.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
us = float(np.median(ts))
if os.environ.get("VTC_TRACE") == "1":
    p.trace()  # reset
    p.execute(s.cuda_stream)
    torch.cuda.synchronize()
    t = p.trace()[0]
    n_ctas = ((S + 127) // 128) * B * H
    blocks = sum(min((S + 127) // 128, qt + 1) for qt in range((S + 127) // 128)) * B * H if causal else n_ctas * ((S + 127) // 128)
    print(json.dumps({"trace_span_us": (int(t[1]) - int(t[0])) / 1e3, "per_kv_block_cycles": {
        "softmax_wait_S": int(t[2]) / blocks, "softmax_wait_PV": int(t[3]) / blocks, "softmax_busy": int(t[4]) / blocks,
        "mma_wait_K": int(t[5]) / blocks, "mma_wait_P": int(t[6]) / blocks, "mma_wait_V": int(t[7]) / blocks}}))
flops = 4.0 * B * H * S * S * 128 * (0.5 if causal else 1.0)
peak = json.load(open(ROOT / "MEASURED_PEAKS.json")).get("bf16_tflops", 1642.6) if (ROOT / "MEASURED_PEAKS.json").exists() else 1642.6
print(json.dumps({"kernel": [l["kernel"] for l in p.info()["launches"]], "us": us, "tflops": flops / us / 1e6,
                  "frac": flops / us / 1e6 / peak, "shape": [B, S, H, HKV], "causal": causal}))

"""Kernel micro-benchmarks (one GPU): single-node VTC graphs timed with CUDA
events over CUDA-graph replays, next to torch reference ops of the same shape.
Used to size individual kernels against their roofline; not the headline bench."""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2604_09558_b200 as vtc  # noqa: E402
from paper_2604_09558_b200.workloads import GraphBuilder  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream()
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
read_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timeit(fn, reps=50, flush=False):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        if flush:
            flush_buf.random_(0, 255)
            read_buf.max()
        else:
            torch.cuda._sleep(20000)  # keep the device busy while the host enqueues
        s.record(stream)
        fn()
        e.record(stream)
        e.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return float(np.median(ts))


def plan_of(doc, flags=0, mode=vtc.MAX_ELIMINATION):
    g = vtc.parse_graph(doc)
    p = vtc.Plan(g, mode, flags=flags)
    # random device inputs
    for tid, t in g.tensors().items():
        if t["kind"] == "input":
            a = torch.randn(t["shape"], device=dev).mul_(0.05).to(torch.bfloat16)
            p.bind_root(tid, a.data_ptr())
            keep.append(a)
    p.prepare()
    return g, p


keep = []
rows = []

# 1. trivial kernels
x = torch.randn(4096, device=dev).to(torch.bfloat16)
rows.append(("torch add [4096] bf16", timeit(lambda: torch.add(x, x))))
gb = GraphBuilder("bf16")
gb.input("a", [1, 32, 128])
gb.input("b", [1, 32, 128])
gb.node("add", "Add", ["a", "b"], "y", out_kind="output")
g, p = plan_of(gb.doc())
rows.append(("vtc eltwise add [1,32,128] (graph replay)", timeit(lambda: p.execute_graph(stream))))
rows.append(("vtc eltwise add [1,32,128] (direct launch)", timeit(lambda: p.execute(stream))))
ms = p.execute_timed(1, stream)
rows.append(("vtc eltwise add event-timed in graph", float(ms[0]) * 1e3))

# 2. GEMV shapes
for K, N in ((4096, 6144), (4096, 4096), (4096, 14336), (14336, 4096)):
    gb = GraphBuilder("bf16")
    gb.input("a", [1, K])
    gb.input("w", [K, N])
    gb.node("mm", "MatMul", ["a", "w"], "y", out_kind="output")
    mb = K * N * 2 / 1e6
    for name, flags in (("stream", 0), ("ldg", 8)):
        try:
            g, p = plan_of(gb.doc(), flags=flags)
            t = timeit(lambda: p.execute_graph(stream), flush=True)
            rows.append((f"vtc gemv[{name}] 1x{K}x{N} ({mb:.0f} MB)", t, mb * 1e6 / (t * 1e-6) / 1e9))
        except Exception as e:  # noqa: BLE001
            rows.append((f"vtc gemv[{name}] 1x{K}x{N}", f"ERR {e}"))
    A = torch.randn(1, K, device=dev).to(torch.bfloat16)
    W = torch.randn(K, N, device=dev).to(torch.bfloat16)
    t = timeit(lambda: torch.matmul(A, W), flush=True)
    rows.append((f"torch matmul 1x{K}x{N}", t, mb * 1e6 / (t * 1e-6) / 1e9))

# 3. copy bandwidth reference
big = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
big2 = torch.empty_like(big)
t = timeit(lambda: big2.copy_(big), reps=20)
rows.append(("torch copy 512MiB", t, 2 * big.numel() / (t * 1e-6) / 1e9))

for r in rows:
    print(" | ".join(str(c) if not isinstance(c, float) else f"{c:.2f}" for c in r))

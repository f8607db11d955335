"""Host<->device round-trip floor on this box: graph replay + sync with and
without 8 KB H2D / D2H memcpy nodes and a tiny kernel (for the e2e budget)."""
import time
import numpy as np
import torch

s = torch.cuda.Stream()
hin = torch.empty(4352, dtype=torch.int16).pin_memory()
hout = torch.empty(4096, dtype=torch.int16).pin_memory()
din = torch.empty_like(hin, device="cuda")
dout = torch.empty_like(hout, device="cuda")


def graph(body):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        body()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            body()
    return g


cases = {
    "kernel only": lambda: dout.add_(1),
    "h2d+kernel+d2h": lambda: (din.copy_(hin, non_blocking=True), dout.add_(1), hout.copy_(dout, non_blocking=True)),
}
for name, body in cases.items():
    g = graph(body)
    for mode in ("event", "wall"):
        ts = []
        for _ in range(200):
            torch.cuda.synchronize()
            if mode == "event":
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(s)
                g.replay()
                s.synchronize()
                b.record(s)
                b.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            else:
                t0 = time.perf_counter()
                g.replay()
                s.synchronize()
                ts.append((time.perf_counter() - t0) * 1e6)
        print(f"{name:18s} {mode:5s} median {np.median(ts):6.1f} us  p10 {np.percentile(ts, 10):6.1f}")

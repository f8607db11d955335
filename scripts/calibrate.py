"""Fit the analytic cost model's MachineParams (proj/include/vtelim/cost_model.hpp:18-28)
to one B200, then check how well estimate() predicts measured plan times.

  bandwidth / kernel_launch_overhead : contiguous gather-copy launches (Reshape
                                       materialised) over 64 KB .. 1 GB, t = L + bytes / BW
  coalesce_unit / partial_penalty    : Slice copies whose contiguous runs are 4 .. 1024 B
  noncoalesced_penalty               : element-scattered Transpose copies (4-byte runs)
  launch overhead inside a graph     : a chain of 32 tiny dependent copies, per launch

Writes gpurun_out/calibration.json (copy to profiles/r2_calibration.json).
Run on the GPU box:  python scripts/calibrate.py
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402  (events and the stream only)

import paper_2604_09558_b200 as vtc  # noqa: E402
from paper_2604_09558_b200 import workloads as W  # noqa: E402
from paper_2604_09558_b200.workloads import GraphBuilder  # noqa: E402


def replay_us(plan, reps=30, warm=5):
    s = torch.cuda.Stream()
    plan.prepare()
    for _ in range(warm):
        plan.execute_graph(s.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        a.record(s)
        plan.execute_graph(s.cuda_stream)
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


def one_copy(kind, n_elems, run=None, dtype="f32"):
    g = GraphBuilder(dtype)
    if kind == "contig":
        g.input("x", [n_elems // 256, 256])
        g.node("dm", "Reshape", ["x"], "y", {"shape": [256, n_elems // 256]}, out_kind="output")
    elif kind == "transpose":
        r = int(np.sqrt(n_elems))
        g.input("x", [r, r])
        g.node("dm", "Transpose", ["x"], "y", {"perm": [1, 0]}, out_kind="output")
    elif kind == "slice":
        cols = 2 * run
        rows = max(1, n_elems // run)
        g.input("x", [rows, cols])
        g.node("dm", "Slice", ["x"], "y", {"axes": [1], "starts": [0], "ends": [run]}, out_kind="output")
    return g.doc()


def chain(n_ops, n_elems=1024):
    g = GraphBuilder("f32")
    g.input("x", [32, n_elems // 32])
    cur, shape = "x", [32, n_elems // 32]
    for i in range(n_ops):
        shape = shape[::-1]
        out = f"t{i}"
        g.node(f"n{i}", "Transpose", [cur], out, {"perm": [1, 0]}, out_kind="output" if i == n_ops - 1 else "intermediate")
        cur = out
    return g.doc()


def measure(doc, mode=vtc.MATERIALIZE):
    g = vtc.parse_graph(doc)
    p = vtc.Plan(g, mode)
    est = g.estimate(None if mode == vtc.MATERIALIZE else p.info(dry=True)["selected"], {"bandwidth": 1.0})
    return replay_us(p), est


def main():
    out = {"device": torch.cuda.get_device_name(0), "points": {}}
    # contiguous copies
    xs, ys = [], []
    for mb in (0.0625, 0.25, 1, 4, 16, 64, 256, 1024):
        n = int(mb * (1 << 20) / 4) // 256 * 256
        t, est = measure(one_copy("contig", n))
        bytes_ = est["total_bytes"]
        xs.append(bytes_)
        ys.append(t)
        out["points"].setdefault("contig", []).append({"bytes": bytes_, "us": t})
    A = np.vstack([np.ones(len(xs)), np.array(xs, float)]).T
    (L, inv_bw), *_ = np.linalg.lstsq(A, np.array(ys), rcond=None)
    big = [(b, t) for b, t in zip(xs, ys) if b >= 64 << 20]
    bw = float(np.median([b / (t - L) for b, t in big]))  # bytes / us, large copies
    # element-scattered transposes
    pen = []
    for mb in (16, 64, 256):
        n = int(mb * (1 << 20) / 4)
        t, est = measure(one_copy("transpose", n))
        out["points"].setdefault("transpose", []).append({"bytes": est["total_bytes"], "us": t})
        # model: reads are non-coalesced, writes contiguous
        half = est["total_bytes"] / 2
        pen.append(max(1.0, (t - L - half / bw) / (half / bw)))
    # partial runs
    runs = {}
    for run in (1, 2, 4, 8, 16, 32, 64, 128, 256):
        n = (64 << 20) // 4
        t, est = measure(one_copy("slice", n, run))
        contig_t = L + est["total_bytes"] / bw
        runs[run * 4] = t / contig_t
        out["points"].setdefault("slice", []).append({"run_bytes": run * 4, "bytes": est["total_bytes"], "us": t,
                                                      "ratio_vs_contiguous": t / contig_t})
    coalesce = next((rb for rb in sorted(runs) if runs[rb] <= 1.25), 1024)
    partial = float(np.median([runs[rb] for rb in runs if rb >= coalesce])) if coalesce < 1024 else 1.0
    # dependent-launch overhead inside a CUDA graph
    t32, _ = measure(chain(32))
    t1, _ = measure(chain(1))
    graph_launch = (t32 - t1) / 31
    params = {"bandwidth": round(bw, 1), "coalesce_unit": int(coalesce),
              "kernel_launch_overhead": round(float(graph_launch), 3),
              "noncoalesced_penalty": round(float(np.median(pen)), 3),
              "partial_penalty": round(max(1.0, partial), 3)}
    out["fit"] = {"standalone_launch_us": float(L), "graph_dependent_launch_us": float(graph_launch),
                  "lstsq_bandwidth_bytes_per_us": float(1 / inv_bw) if inv_bw > 0 else None}
    out["params"] = params
    print(json.dumps(params))

    # validation: modelled vs measured plan times (materialised and VTC plans)
    val = []
    cases = {
        "c1_chain_1024": W.c1_chain(1024),
        "fig11_c3k2_N=102400": W.fig11_yolo_c3k2("f32", N=102400, c=64, cin=128, cout=128),
        "fig9_effvit_B16_N4096": W.fig9_efficientvit_attention("f32", B=16, N=4096, C=128, heads=8),
        "fig6_kv": W.fig6_kv_update("f32", L=4096, heads=32, hd=128, pos=7),
    }
    for name, doc in cases.items():
        g = vtc.parse_graph(doc)
        for mode, label in ((vtc.MATERIALIZE, "materialized"), (vtc.MAX_ELIMINATION, "vtc"), (vtc.GREEDY, "greedy")):
            try:
                p = vtc.Plan(g, mode)
                sel = None if mode == vtc.MATERIALIZE else p.info(dry=True)["selected"]
                est = g.estimate(sel, params)
                t = replay_us(p)
                val.append({"case": name, "plan": label, "measured_us": t, "modelled_us": est["total_time"],
                            "ratio": est["total_time"] / t, "dm_kernels": est["data_movement_kernels"]})
            except Exception as e:  # noqa: BLE001
                val.append({"case": name, "plan": label, "error": str(e)[:200]})
    out["validation"] = val
    # savings: modelled (all-physical - plan) vs measured, per case
    for case in cases:
        rows = {v["plan"]: v for v in val if v["case"] == case and "error" not in v}
        if "materialized" in rows and "vtc" in rows:
            m, v = rows["materialized"], rows["vtc"]
            val.append({"case": case, "plan": "saving", "measured_us": m["measured_us"] - v["measured_us"],
                        "modelled_us": m["modelled_us"] - v["modelled_us"],
                        "ratio": (m["modelled_us"] - v["modelled_us"]) / max(1e-9, m["measured_us"] - v["measured_us"])})
    for v in val:
        print(json.dumps(v))
    Path(ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "calibration.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

"""Benchmark: VTC-planned Llama-3-8B decoder-layer decode step on B200.

Metric (BASELINE.json): decoder-layer latency (us) with HBM GB/s as a fraction
of roofline and the DRAM bytes eliminated versus the materialising executor.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4|c5|c1]
                  [--also c3,c4,c5] [--impl vtc|reference] [--l2 none|flush]

Headline workload: BASELINE configs[1] -- Llama-3-8B decoder layer, decode
step, batch 1, KV length 2048, bf16 (random-init weights uniform(-1,1)/
sqrt(fan_in)).  At N=1 the other configurations (C3 decode B=64 KV 8192, C4
Swin-T block B=64, C5 prefill B=8 S=4096) are measured in the same run and
nested under "configs".  Every timed step is one full layer on the GPU (one
CUDA-graph replay): zero data-movement kernels under the VTC plan.  By default
no L2 flush is needed (every step streams more than the 126 MB L2: weights /
KV / activations); --l2 flush writes + reads 256 MiB between steps, outside
the timed events (also reported as l2_flushed_us).  Kernel times for the
roofline come from the in-graph device timeline of the same plan (first-CTA
entry / last-CTA exit per launch, charged as critical-path shares that add up
to the step).  `e2e` runs the step through vtc_run from pinned host buffers;
decode advances the position every step on one plan / one captured graph.
`--impl reference` times the reference's own CPU executor (oracle/_ref, built
from /root/reference) on the same layer.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

CONFIGS = {
    "c2": dict(B=1, L=2048, workload="llama3-8b-decoder-layer-decode-b1-kv2048"),
    "c3": dict(B=64, L=8192, workload="llama3-8b-decoder-layer-decode-b64-kv8192"),
    "c1": dict(n=1024, workload="reshape-transpose-slice-fp32-matmul-1024"),
    "c5": dict(B=8, S=4096, prefill=True, workload="llama3-8b-decoder-layer-prefill-b8-s4096"),
    "c4": dict(B=64, H=56, swin=True, workload="swin-t-stage1-shifted-window-block-b64-224"),
}
METRIC = "decoder-layer latency (us) & HBM GB/s as % roofline; DRAM bytes eliminated"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[4 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
def build_layer_inputs(doc, cfg, torch, dev):
    """Random-init weights / caches directly on the device; per-step inputs on pinned host."""
    from paper_2604_09558_b200 import workloads as W
    specs = {t["id"]: t for t in doc["tensors"]}
    swin = bool(cfg.get("swin"))
    scales = W.swin_weight_scales() if swin else W.llama_weight_scales()
    host_ids = ("x",) if swin else ("x", "cos", "sin")
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    dev_tensors = {}
    for t in doc["tensors"]:
        tid = t["id"]
        if t["kind"] != "input" or tid in host_ids:
            continue
        if tid == "attn_bias":
            dev_tensors[tid] = torch.from_numpy(W.swin_attn_bias()).to(dev).to(torch.bfloat16).contiguous()
            continue
        x = torch.empty(t["shape"], dtype=torch.float32, device=dev).uniform_(-1.0, 1.0, generator=g)
        dev_tensors[tid] = (x * scales.get(tid, 1.0)).to(torch.bfloat16).contiguous()
    B = cfg["B"]
    rng = np.random.default_rng(2)
    if swin:
        host = {"x": torch.from_numpy(rng.uniform(-1, 1, size=specs["x"]["shape"]).astype(np.float32)).to(torch.bfloat16)}
        return dev_tensors, {k: v.contiguous().pin_memory() for k, v in host.items()}
    if cfg.get("prefill"):
        cos, sin = W.rope_tables_prefill(B, cfg["S"])
        rows = B * cfg["S"]
    else:
        cos, sin = W.rope_tables(B, [cfg["L"] - 1] * B)
        rows = B
    host = {
        "x": torch.from_numpy(rng.uniform(-1, 1, size=(rows, 4096)).astype(np.float32)).to(torch.bfloat16),
        "cos": torch.from_numpy(cos.astype(np.float32)).to(torch.bfloat16),
        "sin": torch.from_numpy(sin.astype(np.float32)).to(torch.bfloat16),
    }
    host = {k: v.contiguous().pin_memory() for k, v in host.items()}
    return dev_tensors, host


def time_steps(fn, steps, torch, stream, flush):
    """Per-step CUDA-event timing on `stream`; L2 flushed before each step, outside the events."""
    times = []
    for _ in range(steps):
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        # the flush is queued ahead of the start event: the host enqueues the
        # step while the device is still flushing, so the timed region starts
        # when the flush ends and contains no host launch latency
        flush()
        s.record(stream)
        fn()
        e.record(stream)
        e.synchronize()
        times.append(s.elapsed_time(e))
    return float(np.mean(times)), times


def _ref_layer_setup(cfg):
    """The layer in the reference's own operator vocabulary (f32; RMSNorm ->
    weight Mul, attention -> QK^T * scale -> .V without softmax: the same data
    movement and GEMM work), planned by the reference (all-physical -- its
    planner cannot compose at KV >= 512) on oracle/_ref."""
    import ref
    from paper_2604_09558_b200 import workloads as W
    if not ref.available():
        return None
    doc = W.llama_decode_layer(B=1, L=cfg["L"], dtype="f32", reference_ops_only=True)
    rg = ref.RefGraph(doc)
    rng = np.random.default_rng(1)
    scales = W.llama_weight_scales()
    x = {}
    for t in doc["tensors"]:
        if t["kind"] == "input":
            x[t["id"]] = (rng.uniform(-1, 1, size=t["shape"]) * scales.get(t["id"], 1.0)).astype(np.float32)
    return rg, rg.plan(), x


def _ref_sample(cfg, runs):
    return (f"{runs} full decoder-layer step(s) for batch row 1 of {cfg['B']}, KV {cfg['L']}, f32, "
            f"reference-ops variant (RMSNorm->Mul, softmax omitted), reference execute(), single thread; "
            f"value = per-row time x {cfg['B']} rows (rows are independent)")


def cpu_reference_layer(cfg, runs=2):
    setup = _ref_layer_setup(cfg)
    if setup is None:
        return None
    rg, plan, x = setup
    ts = [plan.execute(x)[1] / 1e3 for _ in range(runs)]
    v = float(np.median(ts)) * cfg["B"]
    return {"value": v, "unit": "us", "cores": 1, "kind": "reference", "sample": _ref_sample(cfg, runs)}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    if args.config == "c1":
        import ref
        from paper_2604_09558_b200 import workloads as W
        if not ref.available():
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
            return
        rg = ref.RefGraph(W.c1_chain(cfg["n"]))
        x = rg.inputs_random(1)
        plan = rg.plan()
        sample = "full C1 chain + 1024^3 f32 matmul, reference execute (all-physical), single thread"
        scale = 1
    else:
        setup = _ref_layer_setup(cfg)
        if setup is None:
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
            return
        rg, plan, x = setup
        sample = _ref_sample(cfg, args.steps)
        scale = cfg["B"]
    ts = []
    for i in range(args.warmup + args.steps):
        _, ns, _ = plan.execute(x)
        if i >= args.warmup:
            ts.append(ns / 1e3 * scale)
    v = float(np.mean(ts))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "us", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v / 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["workload"]},
            "cpu_baseline": {"value": v, "unit": "us", "cores": 1, "kind": "reference", "sample": sample},
            "e2e": {"value": v, "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def timeline(p, reps, torch, stream, flush):
    """Per-launch device time inside the CUDA-graph replay (plan prepared with
    VTC_TRACE=1: first-CTA entry / last-CTA exit per launch, globaltimer).
    Each launch is charged its critical-path share: from the later of its own
    entry and the previous launch's exit to its exit -- so the shares add up to
    the step and a kernel's PDL wait on its predecessor is not counted twice."""
    acc, total = None, 0.0
    for _ in range(reps):
        p.trace()  # reset the accumulators
        flush()
        p.execute_graph(stream)
        torch.cuda.synchronize()
        tr = p.trace().astype(np.float64)
        ent, ext = tr[:, 0], tr[:, 1]
        rec = (ent > 0) & (ent < 2 ** 62) & (ext > 0)
        t0 = ent[rec].min()
        prev = t0
        share = np.zeros(len(tr))
        for i in range(len(tr)):
            if not rec[i]:
                continue
            share[i] = max(0.0, ext[i] - max(prev, ent[i]))
            prev = max(prev, ext[i])
        total += (prev - t0) / 1e3
        acc = share / 1e3 if acc is None else acc + share / 1e3
    return acc / reps, total / reps  # us


def families(launches, share_us):
    fam = {}
    for l, us in zip(launches, share_us):
        f = fam.setdefault(l["kernel"], {"us": 0.0, "bytes": 0, "launches": 0})
        f["us"] += float(us)
        f["bytes"] += int(l["bytes"])
        f["launches"] += 1
    return fam


def prefill_flops(B, S, D=4096, F=14336, nq=4096, nkv=1024, H=32, hd=128):
    T = B * S
    gemm = 2 * T * D * (nq + 2 * nkv) + 2 * T * nq * D + 2 * 2 * T * D * F + 2 * T * F * D
    attn = 2 * 2 * B * H * (S * (S + 1) // 2) * hd
    return {"gemm_tc_bf16": gemm, "attn_fmha": attn, "attn_prefill": attn}


def measure(name, args, torch, vtc, W, dev, stream, flush, world, rank, comm, local):
    """One configuration: VTC plan (device time, timeline, e2e), the materialising
    comparators on the same kernels, roofline of the dominant kernel family."""
    cfg = CONFIGS[name]
    hbm_peak, tf_peak, peak_src = peaks()
    B = cfg["B"]
    L = cfg.get("L", cfg.get("S", cfg.get("H")))
    swin, prefill = bool(cfg.get("swin")), bool(cfg.get("prefill"))
    decode = not swin and not prefill
    tp = world if (world > 1 and decode and not args.replicas) else 1
    if swin:
        doc = W.swin_block(B=B, H=cfg["H"])
    elif prefill:
        doc = W.llama_prefill_layer(B=B, S=cfg["S"])
    else:
        doc = W.llama_decode_layer(B=B, L=L, tp=tp)
    g = vtc.parse_graph(doc)
    dev_tensors, host = build_layer_inputs(doc, cfg, torch, dev)

    def make(mode, flags=0, trace=False):
        if trace:
            os.environ["VTC_TRACE"] = "1"
        try:
            p = vtc.Plan(g, mode, flags=flags)
            if comm is not None:
                p.set_comm(comm)
            for tid, t in dev_tensors.items():
                p.bind_root(tid, t.data_ptr())
            for tid, t in host.items():
                p.upload_ptr(tid, t.data_ptr(), t.numel() * t.element_size(), stream)
            p.prepare()
        finally:
            os.environ.pop("VTC_TRACE", None)
        return p

    def timed(p, sample_clocks=False):
        for _ in range(max(3, args.warmup)):
            p.execute_graph(stream)
        torch.cuda.synchronize()
        if sample_clocks:
            with ClockSampler(local) as clk:
                ms, _ = time_steps(lambda: p.execute_graph(stream), args.steps, torch, stream, flush)
            return ms, clk.summary()
        ms, _ = time_steps(lambda: p.execute_graph(stream), args.steps, torch, stream, flush)
        return ms, None

    vflags = vtc.FLAG_DYNAMIC_POS if decode else 0
    # ---- the VTC plan: device time of one CUDA-graph replay per step ----
    pv = make(vtc.MAX_ELIMINATION, vflags)
    info = pv.info()
    clk = ClockSampler(local).__enter__()
    lat_ms, _ = timed(pv)
    flushed_ms = None
    if args.l2 == "none":
        l2 = args.l2
        args.l2 = "flush"
        flushed_ms, _ = time_steps(lambda: pv.execute_graph(stream), args.steps, torch, stream, flush)
        args.l2 = l2

    # ---- e2e through vtc_run: the step's inputs from pinned host memory (H2D),
    #      the layer, y back to pinned host memory (D2H); decode advances the
    #      position every step (one plan, one captured graph) ----
    y_host = torch.empty(g.tensors()["y"]["shape"], dtype=torch.bfloat16).pin_memory()
    outs = [("y", y_host.data_ptr(), y_host.numel() * 2)]
    nsteps = max(20, args.warmup) + args.steps
    if decode:
        sets = []
        for i in range(nsteps):
            pos = L - nsteps + i
            cos, sin = W.rope_tables(B, [pos] * B)
            hs = {"x": host["x"],
                  "cos": torch.from_numpy(cos.astype(np.float32)).to(torch.bfloat16).pin_memory(),
                  "sin": torch.from_numpy(sin.astype(np.float32)).to(torch.bfloat16).pin_memory(),
                  "__pos": torch.tensor([pos], dtype=torch.int64).pin_memory()}
            sets.append(pv.host_step([(k, t.data_ptr(), t.numel() * t.element_size()) for k, t in hs.items()],
                                     outs, stream))
        h2d = sum(t.numel() * t.element_size() for t in hs.values())
        it = iter(sets)
        e2e_step = lambda: next(it)()  # noqa: E731
    else:
        e2e_step = pv.host_step([(k, t.data_ptr(), t.numel() * t.element_size()) for k, t in host.items()],
                                outs, stream)
        h2d = sum(t.numel() * t.element_size() for t in host.values())
    # the first host-graph replays run slow (first touches of the pinned staging):
    # warm up past that transient, untimed
    for _ in range(nsteps - args.steps):
        e2e_step()
    e2e_ms, _ = time_steps(e2e_step, args.steps, torch, stream, flush)
    d2h = y_host.numel() * 2
    clk.__exit__(None, None, None)
    clocks = clk.summary()
    if decode:
        pv.set_position(L - 1, stream)  # back to the benchmarked position
    del pv

    # ---- timeline of the same plan (traced build): per-family kernel time ----
    pt = make(vtc.MAX_ELIMINATION, vflags, trace=True)
    share, step_us = timeline(pt, max(3, min(args.steps, 10)), torch, stream, flush)
    launches = pt.info()["launches"]
    del pt
    fam = families(launches, share)

    # ---- materialising comparators on the same kernels ----
    pm = make(vtc.MATERIALIZE)
    minfo = pm.info()
    mat_ms, _ = timed(pm)
    del pm
    strong_ms, sinfo = None, None
    if decode:
        ps = make(vtc.INPLACE_UPDATES)
        sinfo = ps.info()
        strong_ms, _ = timed(ps)
        del ps

    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([lat_ms, e2e_ms, mat_ms, strong_ms or 0.0], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        lat_ms, e2e_ms, mat_ms, strong_ms = t.tolist()
        strong_ms = strong_ms or None

    bytes_step = sum(l["bytes"] for l in launches)
    traffic_file = ROOT / "profiles" / "traffic.json"
    traffic_tab = json.loads(traffic_file.read_text()).get(name, {}) if traffic_file.exists() else {}
    if prefill:
        fl = prefill_flops(B, cfg["S"])
        tens = {k: v for k, v in fam.items() if any(k.startswith(f) for f in fl)}
        dom = max(tens, key=lambda k: tens[k]["us"])
        flops = next(v for f, v in fl.items() if dom.startswith(f))
        ach = flops / (fam[dom]["us"] * 1e-6) / 1e12
        roof = {"bound": "tensor", "achieved": ach, "peak": tf_peak, "unit": "TFLOP/s", "frac": ach / tf_peak,
                "traffic": traffic_tab.get(dom), "kernel": dom, "kernel_launches_per_step": fam[dom]["launches"],
                "algorithmic_flops_per_step": flops, "peak_source": peak_src,
                "kernel_time_source": "in-graph device timeline, critical-path share"}
        # every tensor-core family against the tensor roofline (GEMMs and attention)
        by_kernel = {k: {"achieved_tflops": next(v for f, v in fl.items() if k.startswith(f)) / (tens[k]["us"] * 1e-6) / 1e12,
                         "us": tens[k]["us"]} for k in tens}
        for k in by_kernel:
            by_kernel[k]["frac"] = by_kernel[k]["achieved_tflops"] / tf_peak
        roof["by_kernel"] = by_kernel
    else:
        dom = max(fam, key=lambda k: fam[k]["us"])
        ach = fam[dom]["bytes"] / (fam[dom]["us"] * 1e-6) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                "frac_vs_8tbs": ach / 8000.0, "traffic": traffic_tab.get(dom), "kernel": dom,
                "kernel_launches_per_step": fam[dom]["launches"], "algorithmic_bytes_per_step": fam[dom]["bytes"],
                "peak_source": peak_src, "kernel_time_source": "in-graph device timeline, critical-path share"}
        roof["by_kernel"] = {k: {"achieved_gbs": v["bytes"] / (v["us"] * 1e-6) / 1e9, "us": v["us"],
                                 "frac": v["bytes"] / (v["us"] * 1e-6) / 1e9 / hbm_peak} for k, v in fam.items() if v["us"] > 0}
    out = {
        "metric": METRIC, "value": lat_ms * 1e3, "unit": "us", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": lat_ms, "higher_is_better": False,
        "scaling": "strong" if tp > 1 else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights uniform(-1,1)/sqrt(fan_in), random KV cache / activations)",
        "config": {"workload": cfg["workload"], "batch": B,
                   **({"resolution": 224, "stage1_grid": L, "window": 7, "shift": 3} if swin else
                      {"seq_len": L} if prefill else {"kv_len": L, "pos": L - 1}),
                   "parallelism": (f"tp{tp} (head-sharded; 2 NCCL allreduce of [{B},4096] bf16 per layer)" if tp > 1
                                   else f"replicas x{world}" if world > 1 else "single-gpu"),
                   "l2": ("inputs larger than L2: every step streams %.0f MB (> 126 MB L2) with an L2 evict-first "
                          "policy on weights / KV; no explicit flush" % (bytes_step / 1e6)
                          if args.l2 == "none" else "flushed between timed steps (256 MiB write + 256 MiB read)"),
                   "plan": "VTC max-elimination (all data-movement ops virtual)" + (
                       ", dynamic decode position (one plan / graph for every position)" if decode else ""),
                   "cuda_graph": True},
        "roofline": roof,
        "step_hbm_gbs": bytes_step / (lat_ms * 1e-3) / 1e9,
        "step_hbm_frac": bytes_step / (lat_ms * 1e-3) / 1e9 / hbm_peak,
        "step_hbm_frac_vs_8tbs": bytes_step / (lat_ms * 1e-3) / 1e9 / 8000.0,
        "bytes_per_step": bytes_step,
        "timeline_step_us": step_us,
        "kernel_times_us": {k: round(v["us"], 2) for k, v in fam.items()},
        "launch_timeline": [{"node": l.get("node"), "kernel": l["kernel"], "us": round(float(us), 2),
                             "bytes": int(l["bytes"])} for l, us in zip(launches, share)],
        "materialized_us": mat_ms * 1e3,
        "speedup_vs_materialized": mat_ms / lat_ms,
        "strong_materialized_us": strong_ms * 1e3 if strong_ms else None,
        "speedup_vs_strong_materialized": strong_ms / lat_ms if strong_ms else None,
        "l2_flushed_us": flushed_ms * 1e3 if flushed_ms is not None else None,
        "dram_bytes_eliminated": info["bytes_eliminated"],
        "data_movement_launches": {"virtual": info["data_movement_launches"],
                                   "materialized": minfo["data_movement_launches"],
                                   **({"strong_materialized": sinfo["data_movement_launches"]} if sinfo else {})},
        "e2e": {"value": e2e_ms * 1e3, "unit": "us", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                **({"position": f"advances every step ({L - nsteps}..{L - 1}), same plan and graph"} if decode else {})},
        "gpu_launches": info["kernel_launches"] * args.steps,
        "clocks": clocks,
    }
    if prefill:
        out["tflops"] = sum(prefill_flops(B, cfg["S"]).values()) / (lat_ms * 1e-3) / 1e12
    return out


def run_vtc(args):
    import torch
    import paper_2604_09558_b200 as vtc
    from paper_2604_09558_b200 import workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    read_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def flush():
        if args.l2 == "flush":
            # write a buffer larger than L2, then read another one so the dirty
            # lines are written back here rather than inside the timed step
            flush_buf.random_(0, 255)
            read_buf.max()
        else:
            # inputs larger than L2: no flush; keep the device busy while the
            # host enqueues the step so no launch gap lands inside the events
            torch.cuda._sleep(50000)

    if args.config == "c1":
        hbm_peak, _, peak_src = peaks()
        return run_c1(args, torch, vtc, W, dev, stream, flush, hbm_peak, peak_src, world, rank)
    comm = None
    if world > 1 and not args.replicas:
        import torch.distributed as dist
        uid = [vtc.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = vtc.Comm(uid[0], world, rank)
    line = measure(args.config, args, torch, vtc, W, dev, stream, flush, world, rank, comm, local)
    cfg = CONFIGS[args.config]
    if rank == 0:
        decode = not cfg.get("swin") and not cfg.get("prefill")
        line["cpu_baseline"] = (cpu_reference_layer(cfg) if world == 1 and decode and not os.environ.get("BENCH_NO_CPU")
                                else None)
    # the other BASELINE configurations, measured in the same run (N = 1)
    if world == 1 and args.also:
        nested = {}
        for name in [c for c in args.also.split(",") if c and c != args.config]:
            try:
                nested[name] = measure(name, args, torch, vtc, W, dev, stream, flush, world, rank, None, local)
            except Exception as e:  # report, keep the headline line
                nested[name] = {"error": f"{type(e).__name__}: {e}"}
        line["configs"] = nested
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_c1(args, torch, vtc, W, dev, stream, flush, hbm_peak, peak_src, world, rank):
    import vtc_oracle as O
    doc = W.c1_chain(1024)
    g = vtc.parse_graph(doc)
    x = O.random_inputs(doc, 1)
    res = {}
    for name, mode in (("virtual", vtc.MAX_ELIMINATION), ("materialized", vtc.MATERIALIZE)):
        p = vtc.Plan(g, mode)
        for tid, a in x.items():
            p.upload(tid, a, stream)
        p.prepare()
        for _ in range(max(3, args.warmup)):
            p.execute_graph(stream)
        with ClockSampler(0) as clk:
            res[name], _ = time_steps(lambda: p.execute_graph(stream), args.steps, torch, stream, flush)
        if name == "virtual":
            info = p.info()
            clocks = clk.summary()
    flops = 2 * 1024 ** 3
    line = {"metric": METRIC, "value": res["virtual"] * 1e3, "unit": "us", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["virtual"], "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": CONFIGS["c1"]["workload"], "exact_fp32": True},
            "tflops": flops / (res["virtual"] * 1e-3) / 1e12, "materialized_us": res["materialized"] * 1e3,
            "dram_bytes_eliminated": info["bytes_eliminated"], "clocks": clocks,
            "gpu_launches": info["kernel_launches"] * args.steps}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="vtc", choices=["vtc", "reference"])
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent full layers instead of head sharding")
    ap.add_argument("--also", default="c3,c4,c5",
                    help="other configurations measured in the same run and nested under 'configs' (N=1; '' = none)")
    ap.add_argument("--l2", default="none", choices=["flush", "none"],
                    help="flush L2 between timed steps, or rely on the step's inputs exceeding L2")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_vtc(args)


if __name__ == "__main__":
    main()

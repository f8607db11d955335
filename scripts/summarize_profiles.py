"""Turn the ncu outputs of scripts/profile_round.sh (gpurun_out/) into the
tracked summaries under profiles/: per-launch tables of the vtc kernels of one
decode step (device time, DRAM bytes) and profiles/traffic.json (measured DRAM
bytes per launch of each kernel family, read by bench.py for roofline.traffic)."""
import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
TAG = sys.argv[1] if len(sys.argv) > 1 else "r1"
FAMILY = {"gemv_stream_kernel": "gemv_stream_bf16", "gemv_kernel": "gemv_bf16", "attn_decode_kernel": "attn_decode_tc_splitkv",
          "combine_fast_kernel": "attn_decode_tc_splitkv", "ew_flat_kernel": "eltwise_flat", "ew_kernel": "eltwise",
          "row_kernel": "rowop", "row_warp_kernel": "rowop", "row_vec_kernel": "rowop", "row_long_kernel": "rowop",
          "gemm_tc_kernel": "gemm_tc_bf16", "mm_kernel": "matmul_tiled", "attn_prefill_kernel": "attn_prefill_tc",
          "attn_kernel": "attention", "host_link_copy_kernel": "host_link_copy"}


def family(name):
    for k, v in FAMILY.items():
        if k in name:
            return v
    return None


def launches(cfg):
    d = defaultdict(dict)
    names = {}
    for fn in (f"launches_{cfg}.csv", f"dram_{cfg}.csv"):  # time pass, DRAM-bytes pass (same launch ids)
        if not (OUT / fn).exists():
            continue
        rows = list(csv.reader(open(OUT / fn)))
        hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
        h = rows[hi]
        ii, ki, mi, vi = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
        ui = h.index("Metric Unit") if "Metric Unit" in h else None
        for r in rows[hi + 1:]:
            v = float(r[vi].replace(",", ""))
            unit = r[ui] if ui is not None else ""
            v *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e3, "msecond": 1e6}.get(unit, 1.0)
            d[int(r[ii])][r[mi]] = v
            names[int(r[ii])] = r[ki]
    for i in d:
        d[i].setdefault("dram__bytes_read.sum", 0.0)
        d[i].setdefault("dram__bytes_write.sum", 0.0)
    out = []
    for i in sorted(d):
        fam = family(names[i])
        if fam is None:
            continue
        out.append(dict(id=i, kernel=names[i].split("(")[0].replace("void vtc::<unnamed>::", ""), family=fam,
                        us=d[i]["gpu__time_duration.sum"] / 1e3, read_MB=d[i]["dram__bytes_read.sum"] / 1e6,
                        write_MB=d[i]["dram__bytes_write.sum"] / 1e6))
    return out


def last_step(ls, is_start):
    """The launches of the last complete decode step of the VTC (virtual) plan:
    between two consecutive launches that start a step."""
    starts = [k for k in range(len(ls)) if is_start(ls, k)]
    for a, b in zip(starts[::-1][1:], starts[::-1]):
        if not any(l["kernel"].startswith("ew_kernel") and l["read_MB"] > 100 for l in ls[a:b]):
            step = ls[a:b]
            if not any("gather" in l["kernel"] for l in step):
                return step
    return ls


def c2_start(ls, k):  # the RMSNorm+QKV GEMV (50 MB of weights) opens a C2 step
    return ls[k]["family"].startswith("gemv") and 45 < ls[k]["read_MB"] < 56


def c3_start(ls, k):  # ln1 (rowop) followed by the QKV GEMM opens a C3 step
    return ls[k]["family"] == "rowop" and k + 1 < len(ls) and ls[k + 1]["family"] == "gemm_tc_bf16" and \
        45 < ls[k + 1]["read_MB"] < 60


def c4_start(ls, k):  # ln1 (rowop) followed by the QKV GEMM opens a C4 (Swin) step
    return ls[k]["family"] == "rowop" and k + 2 < len(ls) and ls[k + 1]["family"] == "gemm_tc_bf16" and \
        ls[k + 2]["family"] == "attn_prefill_tc"


traffic = {}
md = [f"# Round {TAG[1:]} ncu summaries (B200, `--clock-control none`, serialized cold-cache launches)\n"]
for cfg, first in (("c2", c2_start), ("c3", c3_start), ("c4", c4_start)):
    p = OUT / f"launches_{cfg}.csv"
    if not p.exists():
        continue
    ls = launches(cfg)
    with open(PROF / f"{TAG}_{cfg}_launches.csv", "w") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "family", "gpu_time_us", "dram_read_MB", "dram_write_MB"])
        for l in ls:
            w.writerow([l["id"], l["kernel"], l["family"], f"{l['us']:.2f}", f"{l['read_MB']:.3f}", f"{l['write_MB']:.3f}"])
    # one virtual-plan step: from the second-to-last to the last occurrence of the step's first kernel
    step = last_step(ls, first)
    fam = defaultdict(lambda: dict(us=0.0, bytes=0.0, n=0))
    for l in step:
        f = fam[l["family"]]
        f["us"] += l["us"]
        f["bytes"] += (l["read_MB"] + l["write_MB"]) * 1e6
        f["n"] += 1
    tot = sum(f["us"] for f in fam.values())
    traffic[cfg] = {k: v["bytes"] / v["n"] for k, v in fam.items()}
    md.append(f"\n## {cfg}: one decode step, {len(step)} vtc launches, sum of serialized launch times {tot:.1f} us\n")
    md.append("| kernel family | launches | ncu time (us) | share | DRAM bytes / launch (MB) |\n|---|---|---|---|---|\n")
    for k, v in sorted(fam.items(), key=lambda kv: -kv[1]["us"]):
        md.append(f"| {k} | {v['n']} | {v['us']:.1f} | {100 * v['us'] / tot:.0f}% | {v['bytes'] / v['n'] / 1e6:.2f} |\n")
(PROF / "traffic.json").write_text(json.dumps(traffic, indent=1))
for rep, label in (("full_gemv_stream", "gemv_stream (C2, 4 launches)"), ("full_attn_c3", "attn_decode (C3)")):
    f = OUT / f"{rep}.ncu-rep"
    if not f.exists():
        continue
    raw = subprocess.run(["ncu", "-i", str(f), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_active.avg",
            "launch__grid_size", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
    md.append(f"\n## `ncu --set full`: {label}\n\n| metric | " + " | ".join(f"launch {i}" for i in range(len(rows) - 2)) + " |\n")
    md.append("|---|" + "---|" * (len(rows) - 2) + "\n")
    for k in keys:
        if k in h:
            j = h.index(k)
            md.append(f"| {k} ({rows[1][j]}) | " + " | ".join(r[j] for r in rows[2:]) + " |\n")
(PROF / f"{TAG}_summary.md").write_text("".join(md))
print("".join(md))

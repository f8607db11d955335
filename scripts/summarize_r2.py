"""Turn the outputs of scripts/profile_r2.sh (gpurun_out/r2_*) into the tracked
summaries under profiles/: per-launch tables of one step of every config
(ncu device time and DRAM bytes per vtc launch, mapped to the plan's nodes),
the --set full metrics of the dominant kernels (tensor-pipe activity for the
tcgen05 GEMMs and attention), the compute-sanitizer verdicts, and
profiles/traffic.json (DRAM bytes per launch of each kernel family; bench.py
reads it for roofline.traffic)."""
import ast
import csv
import json
import re
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"
TAG = sys.argv[1] if len(sys.argv) > 1 else "r2"
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}


def ncu_rows(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ii, ki, mi, vi = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    ui = h.index("Metric Unit") if "Metric Unit" in h else None
    d, names = defaultdict(dict), {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui] if ui is not None else "", 1.0)
        d[int(r[ii])][r[mi]] = v
        names[int(r[ii])] = r[ki]
    return [(i, names[i], d[i]) for i in sorted(d)]


def step_launches(cfg):
    log = OUT / f"{TAG}_launch_{cfg}.log"
    csvp = OUT / f"{TAG}_launch_{cfg}.csv"
    if not (log.exists() and csvp.exists()):
        return None
    plan = None
    for line in log.read_text().splitlines():
        if line.startswith("["):
            plan = ast.literal_eval(line)
            break
    if plan is None:
        return None
    vtc = [r for r in ncu_rows(csvp) if "vtc::" in r[1]]
    step = vtc[len(vtc) // 2:]  # run_plan.py ran the plan twice: the second step
    out = []
    for i, name, m in step:
        short = re.sub(r"\(.*", "", name).replace("void vtc::<unnamed>::", "").replace("vtc::<unnamed>::", "")
        rec = dict(ncu_kernel=short, us=m.get("gpu__time_duration.sum", 0.0) / 1e3,
                   read_MB=m.get("dram__bytes_read.sum", 0.0) / 1e6, write_MB=m.get("dram__bytes_write.sum", 0.0) / 1e6)
        if short.startswith("combine") and out:  # the split-KV combine belongs to the attention launch
            for k in ("us", "read_MB", "write_MB"):
                out[-1][k] += rec[k]
            out[-1]["ncu_kernel"] += "+" + short
            continue
        out.append(rec)
    if len(out) != len(plan):
        print(f"{cfg}: {len(out)} kernels vs {len(plan)} plan launches", file=sys.stderr)
    for rec, entry in zip(out, plan):
        rec["node"], rec["kernel"] = entry.rsplit(":", 1)
    return out[:len(plan)]


md = [f"# Round {TAG[1:]} ncu summaries (B200, `--clock-control none`, serialised cold-cache launches, `VTC_NO_PDL=1`)\n\n"
      "One step of each configuration's VTC plan (`scripts/run_plan.py`, second of two steps). Device times here are "
      "serialised single-kernel times under the profiler; the bench's in-graph timeline (PDL overlap) is the number "
      "that adds up to the step.\n"]
traffic = {}
for cfg in ("c2", "c3", "c4", "c5"):
    ls = step_launches(cfg)
    if not ls:
        continue
    with open(PROF / f"{TAG}_{cfg}_launches.csv", "w") as f:
        w = csv.writer(f)
        w.writerow(["node", "kernel", "ncu_kernel", "gpu_time_us", "dram_read_MB", "dram_write_MB"])
        for l in ls:
            w.writerow([l["node"], l["kernel"], l["ncu_kernel"], f"{l['us']:.2f}", f"{l['read_MB']:.3f}", f"{l['write_MB']:.3f}"])
    tot = sum(l["us"] for l in ls)
    fam = defaultdict(lambda: dict(us=0.0, bytes=0.0, n=0))
    for l in ls:
        f = fam[l["kernel"]]
        f["us"] += l["us"]
        f["bytes"] += (l["read_MB"] + l["write_MB"]) * 1e6
        f["n"] += 1
    traffic[cfg] = {k: v["bytes"] / v["n"] for k, v in fam.items()}
    md.append(f"\n## {cfg}: {len(ls)} launches, sum of serialised launch times {tot:.1f} us\n\n")
    md.append("| node | kernel | ncu time (us) | share | DRAM read (MB) | DRAM write (MB) | DRAM TB/s |\n|---|---|---|---|---|---|---|\n")
    for l in ls:
        tbs = (l["read_MB"] + l["write_MB"]) / l["us"] if l["us"] > 0 else 0.0  # MB / us = TB/s
        md.append(f"| {l['node'][:48]} | {l['kernel']} | {l['us']:.1f} | {100 * l['us'] / tot:.0f}% | {l['read_MB']:.1f} | "
                  f"{l['write_MB']:.1f} | {tbs:.2f} |\n")
(PROF / "traffic.json").write_text(json.dumps(traffic, indent=1))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "smsp__inst_executed.sum"]
for rep, label in (("c2_gemv", "C2 streamed GEMVs (QKV+RoPE, O, gate/up, down)"), ("c3_gemm", "C3 tcgen05 GEMMs"),
                   ("c3_attn", "C3 split-KV decode attention"), ("c4_skinny", "C4 persistent shallow-K GEMMs (QKV, proj, fc1, fc2)"),
                   ("c4_attn", "C4 window attention"), ("c5_gemm", "C5 tcgen05 GEMMs (QKV, O, SwiGLU, down)"),
                   ("c5_attn", "C5 tcgen05 flash attention")):
    f = OUT / f"{TAG}_full_{rep}.ncu-rep"
    if not f.exists():
        continue
    raw = subprocess.run(["ncu", "-i", str(f), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        continue
    h = rows[0]
    md.append(f"\n## `ncu --set full`: {label}\n\n| metric | " + " | ".join(f"launch {i}" for i in range(len(rows) - 2)) + " |\n")
    md.append("|---|" + "---|" * (len(rows) - 2) + "\n")
    for k in KEYS:
        if k in h:
            j = h.index(k)
            md.append(f"| {k} ({rows[1][j]}) | " + " | ".join(r[j] for r in rows[2:]) + " |\n")

md.append("\n## compute-sanitizer\n\n")
for tool in ("memcheck", "racecheck", "synccheck"):
    f = OUT / f"{TAG}_san_{tool}.log"
    if not f.exists():
        continue
    txt = f.read_text()
    summ = [l for l in txt.splitlines() if "ERROR SUMMARY" in l or "RACECHECK SUMMARY" in l]
    res = [l for l in txt.splitlines() if re.search(r"\d+ passed|failed", l)]
    md.append(f"* **{tool}**: {summ[-1].strip() if summ else 'no summary line'}; pytest: {res[-1].strip() if res else '?'}\n")
(PROF / f"{TAG}_summary.md").write_text("".join(md))
print("".join(md))

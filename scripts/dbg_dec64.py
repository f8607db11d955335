import os, sys, subprocess, json
import numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'oracle'); sys.path.insert(0,'tests')
import paper_2604_09558_b200 as vtc, vtc_oracle as oracle
from paper_2604_09558_b200 import workloads as W
from test_gpu import _llama_inputs
cfg = dict(B=64, L=256, pos=200, D=1024, Hq=8, Hkv=2, hd=128, F=2048)
doc = W.llama_decode_layer(**cfg)
x = _llama_inputs(oracle, W, doc, cfg["B"], cfg["pos"], cfg["D"], cfg["F"], cfg["hd"])
g = vtc.parse_graph(doc)
outs = {}
for name, envs in [("default", {}), ("noaff", {"VTC_NO_EW_AFF": "1"}), ("nofast", {"VTC_NO_EW_FAST": "1"}), ("norow", {"VTC_NO_ROW_FAST": "1"}), ("default2", {})]:
    for k in ("VTC_NO_EW_AFF", "VTC_NO_EW_FAST", "VTC_NO_ROW_FAST"): os.environ.pop(k, None)
    os.environ.update(envs)
    p = vtc.Plan(g, vtc.MAX_ELIMINATION)
    outs[name] = vtc.execute(g, p, x)["y"]
    print(name, [l['kernel'] for l in p.info()['launches']])
for n in outs: print(n, np.array_equal(outs[n], outs["default"]), int((outs[n] != outs['default']).sum()))

"""Head-sharded (tensor-parallel) decoder layer: host-side logic on CPU.

SURVEY.md §8 e: each rank owns Hq/N query heads, Hkv/N KV heads and F/N FFN
columns; exactly two AllReduce(sum) nodes (after O-proj, after FFN-down) are
the only exchange.  These tests run the per-rank graphs with the CPU oracle in
world_size-2 `gloo` process groups and check that the sharded layer equals the
unsharded one, and that every rank's VTC plan has zero data-movement kernels
and exactly two collectives (the plan is built dry: no GPU needed).
"""
import os
import socket
import sys
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = dict(B=2, L=48, pos=30, D=256, Hq=4, Hkv=2, hd=64, F=512)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _full_inputs():
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import vtc_oracle as O
    from paper_2604_09558_b200 import workloads as W
    doc = W.llama_decode_layer(**CFG)
    x = O.random_inputs(doc, seed=11, scales=W.llama_weight_scales(CFG["D"], CFG["F"]))
    cos, sin = W.rope_tables(CFG["B"], [CFG["pos"]] * CFG["B"], hd=CFG["hd"])
    x["cos"] = O.f32_to_bf16(cos.astype(np.float32))
    x["sin"] = O.f32_to_bf16(sin.astype(np.float32))
    return doc, x


def _rank_main(rank, world, port, outdir):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import vtc_oracle as O
    from paper_2604_09558_b200 import workloads as W
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    _, full = _full_inputs()
    doc = W.llama_decode_layer(**CFG, tp=world)
    mine = W.shard_llama_inputs(full, rank, world, Hq=CFG["Hq"], Hkv=CFG["Hkv"], hd=CFG["hd"], F=CFG["F"])

    def allreduce(v):
        t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.numpy()

    env = O.execute(doc, mine, keep_all=True, allreduce=allreduce)
    np.save(os.path.join(outdir, f"y{rank}.npy"), env["y"])
    np.save(os.path.join(outdir, f"kc{rank}.npy"), env["k_r"])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_head_sharded_layer_equals_unsharded_gloo(oracle, world):
    import torch.multiprocessing as mp
    doc, full = _full_inputs()
    want = oracle.execute(doc, full, keep_all=True)
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank_main, args=(world, _free_port(), d), nprocs=world, join=True)
        ys = [np.load(os.path.join(d, f"y{r}.npy")) for r in range(world)]
        kr = [np.load(os.path.join(d, f"kc{r}.npy")) for r in range(world)]
    # every rank holds the same (allreduced) output ...
    for r in range(1, world):
        assert np.array_equal(ys[r], ys[0])
    got = oracle.bf16_to_f32(ys[0]).astype(np.float64)
    ref = oracle.bf16_to_f32(want["y"]).astype(np.float64)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 2e-2
    # ... and the roped K rows of its own KV heads, bit for bit (no exchange before attention)
    hk = CFG["Hkv"] // world
    for r in range(world):
        assert np.array_equal(kr[r], want["k_r"][:, r * hk:(r + 1) * hk, :])


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_plans_have_two_collectives_and_no_dm_kernels(vtc, world):
    from paper_2604_09558_b200 import workloads as W
    doc = W.llama_decode_layer(B=64, L=8192, tp=world)
    g = vtc.parse_graph(doc)
    info = vtc.Plan(g, vtc.MAX_ELIMINATION).info(dry=True)
    kinds = [l["kernel"] for l in info["launches"]]
    assert info["data_movement_launches"] == 0
    assert kinds.count("allreduce_nccl") == 2
    # the per-rank KV cache is 1/world of the full cache
    kc = [t for t in doc["tensors"] if t["id"] == "k_cache"][0]
    assert kc["shape"] == [8192, 64, 8 // world, 128]

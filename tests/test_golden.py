"""The numpy oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py runs the unmodified vtelim library): every
data-movement operator in f64 / f32 / i64, the C1 chain and the paper's
frame-2 chain, bit for bit.  Needs neither /root/reference nor a GPU."""
import json
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"


def golden_cases():
    index = json.loads((GOLD / "ref_small.json").read_text())
    arrays = np.load(GOLD / "ref_small.npz")
    for name in sorted(index):
        ins = {k: arrays[f"{name}/in/{k}"] for k in index[name]["inputs"]}
        outs = {k: arrays[f"{name}/out/{k}"] for k in index[name]["outputs"]}
        yield name, index[name]["doc"], ins, outs


def fnv1a64(a):
    h = 1469598103934665603
    for b in np.ascontiguousarray(a).view(np.uint8).tobytes():
        h = ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


CASES = list(golden_cases())


@pytest.mark.parametrize("name,doc,ins,outs", CASES, ids=[c[0] for c in CASES])
def test_oracle_matches_reference_golden(oracle, name, doc, ins, outs):
    got = oracle.execute(doc, ins)
    for k, want in outs.items():
        assert got[k].dtype == want.dtype and got[k].shape == want.shape, k
        assert np.array_equal(got[k].view(np.uint8), np.ascontiguousarray(want).view(np.uint8)), (name, k)


def test_golden_digest_matches_survey():
    dig = json.loads((GOLD / "ref_digests.json").read_text())
    assert dig["c1_chain_1024_f32_seed1"]["y"] == "fc294cee5f1ab03e"  # SURVEY.md §8 c

"""Pin the CPU oracle (oracle/paste_oracle.c) to the reference's own outputs.

The golden vectors were produced by running the reference implementation
(tests/golden/make_golden.py).  Here the packing / decoding of this package
plus the oracle must reproduce them exactly; the GPU tests then compare the
CUDA kernels with this pinned oracle.
"""

import numpy as np
import pytest

import golden_io as G
from oracle import bridge
from paper_2603_18897_b200.packing import (PoolImage, SigTable, admit_tables, decode_actions,
                                           decode_predictions, pack_windows)
from paper_2603_18897_b200.tape import KeyTable

CASES = G.golden("predict_golden.json")["cases"]


def run_oracle_case(case, threads=1):
    pool = G.pool(case["pool"])
    sigs, keys = SigTable(), KeyTable()
    image = PoolImage.compile(pool, sigs, keys)
    windows = [[G.event(e) for e in w] for w in case["windows"]]
    batch = pack_windows(windows, sigs, keys, capacity=16)
    K = case["max_candidates"] or max(image.max_bucket, 1)
    pol = G.policy(case["policy"])
    tables = None
    if pol is not None:
        book = G.estimates(case["estimates"])
        tables = admit_tables(sigs, pol, book.duration)
    res = bridge.predict(image, batch, K, tables, threads=threads)
    preds = decode_predictions(res, image, batch.arena, batch.created, None)
    acts = decode_actions(res, preds) if pol is not None else None
    return preds, acts, res


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_predict_matches_reference(case):
    preds, acts, res = run_oracle_case(case)
    assert len(preds) == len(case["expected"])
    for got, exp in zip(preds, case["expected"]):
        assert G.same([G.pred_dict(p) for p in got], exp)
    assert int(res.struct_err.sum()) == case["structural_errors"]
    if acts is not None:
        for s, (got, exp) in enumerate(zip(acts, case["expected_actions"])):
            assert [(preds[s].index(a.prediction), int(a.level), a.expected_utility)
                    for a in got] == [(e["pred"], e["level"], e["utility"]) for e in exp]


def test_oracle_threads_agree():
    case = next(c for c in CASES if c["name"] == "stress_K8")
    a = run_oracle_case(case, threads=1)[2]
    b = run_oracle_case(case, threads=4)[2]
    for f in ("n_pred", "pred_pat", "pred_comp", "n_act", "act_pred", "act_util"):
        assert np.array_equal(getattr(a, f), getattr(b, f))

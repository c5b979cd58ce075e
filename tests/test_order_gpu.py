"""K1 general path on the device (csrc/order.cu, paste_ingest_order):
ingest_trace's grouping, stable (t_start, seq) sort, reorder tally and gap
split (events.py:196-252) == the REFERENCE's ingest output on every ingest
golden, == the pinned oracle (oracle/order.py) on large interleaved traces
with long sessions (CTA sort + merge passes), and mine_columnar over an
unsorted trace == mine_columnar over the same trace pre-ordered."""

import numpy as np
import pytest
import torch

from golden_io import golden
from oracle.order import order_trace
from order_cases import random_trace, raw_columns
from paper_2603_18897_b200._native import PasteUnsupported
from paper_2603_18897_b200.mine_engine import order_columnar
from test_ingest_golden import expected_columns

pytestmark = pytest.mark.gpu
CASES = golden("ingest_golden.json")["cases"]
KEYS = ("session", "seq", "t_start", "t_end", "sig")


def _dev(c):
    return {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in c.items()}


def _check(got, cols, n_seg, reord, order=None):
    for k in KEYS:
        assert np.array_equal(got.columns[k].cpu().numpy(), cols[k]), k
    assert got.n_segments == n_seg
    assert got.reordered_sessions == reord
    if order is not None:
        assert np.array_equal(got.order.cpu().numpy(), order)


@pytest.mark.parametrize("i", range(len(CASES)))
def test_device_order_equals_reference_ingest(i):
    case = CASES[i]
    raw, n_sess = raw_columns(case)
    thr = 300_000.0 if case["threshold"] is None else case["threshold"]
    got = order_columnar(_dev(raw), n_sess, thr)
    exp, _tools, n_seg = expected_columns(case)
    _check(got, exp, n_seg, case["expected"]["reordered"])


@pytest.mark.parametrize("interleave,long_sessions,n_sess", [
    (False, (), 50_000),                      # grouped: identity placement, warp path
    (True, (), 50_000),                       # interleaved: scatter + arrival ranks
    (False, (33, 100, 2048, 2049, 9000), 20_000),  # CTA path: one chunk, chunks + merges
    (True, (64, 5000, 20_000), 20_000),
])
def test_device_order_equals_oracle(interleave, long_sessions, n_sess):
    raw = random_trace(n_sess, seed=len(long_sessions) * 2 + interleave,
                       long_sessions=long_sessions, interleave=interleave)
    got = order_columnar(_dev(raw), n_sess, 300_000.0, with_order=True)
    cols, n_seg, reord, order = order_trace(*(raw[k] for k in KEYS), n_sess, 300_000.0)
    assert reord > 0 and n_seg > n_sess
    _check(got, cols, n_seg, reord, order)


def test_device_order_unused_ids_and_empty():
    raw = random_trace(1000, seed=3, interleave=True)
    raw["session"] = raw["session"] * 3 + 1  # ids 0, 2, 3, 5, ... unused
    got = order_columnar(_dev(raw), 3000, 1000.0)
    cols, n_seg, reord, _ = order_trace(*(raw[k] for k in KEYS), 3000, 1000.0)
    _check(got, cols, n_seg, reord)
    empty = {k: v[:0] for k, v in raw.items()}
    got = order_columnar(_dev(empty), 5, 1000.0)
    assert got.n_segments == 0 and got.columns["sig"].numel() == 0


def test_device_order_rejects_nan_and_bad_ids():
    raw = random_trace(200, seed=4)
    raw["t_start"][17] = np.nan
    with pytest.raises(PasteUnsupported):
        order_columnar(_dev(raw), 200, 300_000.0)
    raw = random_trace(200, seed=4)
    with pytest.raises(ValueError):
        order_columnar(_dev(raw), 100, 300_000.0)


def test_mine_columnar_orders_unsorted_traces():
    """An unsorted / interleaved columnar trace no longer raises: the count
    runs over the device-ordered segments and equals the count of the trace
    ordered up front."""
    from paper_2603_18897_b200.mine_engine import mine_columnar
    from paper_2603_18897_b200.mining import MiningConfig
    from paper_2603_18897_b200.packing import SigTable
    from paper_2603_18897_b200.synth import C4_TOOLS, columnar_corpus

    c = columnar_corpus(300_000, seed=13)
    perm = np.random.default_rng(1).permutation(len(c["sig"]))
    shuffled = {k: v[perm] for k, v in c.items()}
    sigs = SigTable(C4_TOOLS)
    cfg = MiningConfig(k=3, sigma=5, tau=0.3)
    got = mine_columnar(_dev(shuffled), sigs, cfg)
    cols, _, _, _ = order_trace(*(shuffled[k] for k in KEYS), int(c["session"].max()) + 1,
                                300_000.0)
    exp = mine_columnar(_dev(cols), sigs, cfg, inactivity_ms=float("inf"))
    assert got == exp and len(got) > 0
    assert mine_columnar(_dev(c), sigs, cfg) == exp

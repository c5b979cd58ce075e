"""The K1 general-path oracle (oracle/order.py) pinned to the REFERENCE's
ingest_trace output on every ingest golden (tests/golden/ingest_golden.json):
same tool events in order, segment numbering, sigs, segment count and
reordered-session tally."""

import numpy as np
import pytest

from golden_io import golden
from oracle.order import order_trace
from order_cases import raw_columns
from test_ingest_golden import expected_columns

CASES = golden("ingest_golden.json")["cases"]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_order_oracle_equals_reference_ingest(i):
    case = CASES[i]
    raw, n_sess = raw_columns(case)
    thr = 300_000.0 if case["threshold"] is None else case["threshold"]
    cols, n_seg, reord, _ = order_trace(*(raw[k] for k in ("session", "seq", "t_start", "t_end",
                                                           "sig")), n_sess, thr)
    exp, _tools, exp_seg = expected_columns(case)
    for k in exp:
        assert np.array_equal(cols[k], exp[k]), k
    assert n_seg == exp_seg
    assert reord == case["expected"]["reordered"]

"""CompactRecords.expand on hand-built streams (host logic, no device):
the PASTE_CF_ENTRY16 serving format (prediction list = match-table entry,
completeness from the arg stream) expands to the same records as the
per-prediction code stream."""
import numpy as np

from paper_2603_18897_b200._native import (PASTE_CF_ARG16, PASTE_CF_ENTRY16, PASTE_CF_HDR8,
                                           PASTE_CF_PRED8, PATTERN_DTYPE)
from paper_2603_18897_b200.live import CompactRecords


def _patterns():
    pats = np.zeros(4, PATTERN_DTYPE)
    pats["target_tool"] = [0, 1, 2, 1]
    pats["n_bind"] = [1, 0, 2, 1]
    pats["flags"] = [1, 0, 1, 1]  # bit 0 = has mapping
    pats["p"] = [0.9, 0.8, 0.5, 0.25]
    return pats


def test_entry16_expands_like_the_code_stream():
    pats = _patterns()
    benefit = np.array([100.0, 20.0, 7.0])
    K, B, n = 3, 2, 4
    # match table: key -> first records (pattern ids); n_match per key
    entries = (np.array([3, 1, 0, 2], np.int32),
               np.array([[0, 2, 1], [3, 0, 0], [0, 0, 0], [2, 3, 0]], np.int32))
    keys = np.array([0, 1, 0xFFFF, 3], np.uint16)  # session 2: no entry
    n_pred = np.array([3, 1, 0, 2])
    n_act = np.array([2, 1, 0, 1])
    hdr = (n_pred | (n_act << 4)).astype(np.uint8)
    # args in session / rank / binding order: s0: p0 (1), p2 (2, one
    # unresolved) | s1: p3 (1) | s3: p2 (2), p3 (1, unresolved)
    arg = np.array([(1 << 11) | 5, 7, 0xFFFF, 9, 11, 12, 0xFFFF], np.uint16)
    act = np.array([0 | (3 << 5), 2 | (1 << 5), 0 | (2 << 5), 1 | (1 << 5)], np.uint8)
    comp = {0: [0, 1, 2], 1: [0], 3: [0, 1]}  # FULL, PARTIAL, TOOL_ONLY
    code = []
    for s in range(n):
        for i in range(n_pred[s]):
            code.append(entries[1][keys[s], i] | (comp[s][i] << 6))
    fmt = PASTE_CF_HDR8 | PASTE_CF_PRED8 | PASTE_CF_ARG16
    a = CompactRecords(K, B, hdr, np.array(code, np.uint8), arg, act, fmt).expand(pats, benefit)
    b = CompactRecords(K, B, hdr, keys, arg, act, fmt | PASTE_CF_ENTRY16, entries).expand(
        pats, benefit)
    for f in ("n_pred", "n_act", "pred_pat", "pred_comp", "pred_arg", "act_pred", "act_level"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(a.act_util.view(np.int64), b.act_util.view(np.int64))
    assert b.pred_comp[0 * K + 1] == 1 and b.pred_comp[0 * K + 2] == 2
    assert b.pred_arg[(1 * K + 0) * B] == (1 << 32) | 9

"""Host side of the serving wire, on CPU: the packed narrow input layouts
(EventBatch.narrowed, wire8_layout), the key-stream buffer layout
(keys_layout) and CompactRecords.expand of a key + unit-reference download
(PASTE_CF_KEYS | PASTE_CF_UNIQ) against hand-built plan entries -- bindings
that share a resolution unit, an unresolved unit making its predictions
PARTIAL and their admitted actions take the partial level, and a session
without an entry; and the u8 plan-code key stream (PASTE_CF_KEY8): the
codes plan_codes assigns and the same expansion through them."""

import numpy as np

from paper_2603_18897_b200 import _native
import pytest

from paper_2603_18897_b200.live import (CompactRecords, EventBatch, EventCodes, NodeCodes,
                                         keys_layout, plan_codes,
                                         plan_layout_host, wire8_layout)
from paper_2603_18897_b200.packing import C_FULL, C_PARTIAL, C_TOOL_ONLY


def test_narrow_wire_layouts():
    n = 37
    tok = np.arange(n, dtype=np.int32) % 7
    tok[3] = -1  # an LLM step
    node = (np.arange(n, dtype=np.int32) * 11) % 500
    ref = np.stack([node.astype(np.int64), np.zeros(n, np.int64)], axis=1)
    b = EventBatch(tok, ref, np.zeros(1, np.uint8), node).narrowed()
    off, size = wire8_layout(n)
    assert off % 16 == 0 and off >= n and size == off + 2 * n
    assert b.packed.size == size and b.node8 is None
    assert np.array_equal(b.tok8, np.where(tok < 0, 255, tok))
    assert np.array_equal(b.packed[:n], b.tok8)
    assert np.array_equal(b.packed[off:off + 2 * n].view(np.uint16), node)
    assert b.wire(False, narrow8=True)[0] is b.packed
    # values that do not fit keep the wide forms
    big = EventBatch(tok, ref, np.zeros(1, np.uint8), node + 70_000).narrowed()
    assert big.tok8 is None and big.packed is None


def test_event_codes_one_byte_form():
    """(token, node array) pairs -> u8 event codes: append-only, the decode
    table holds (token, node_base) with -1 for an LLM step, and past 256
    pairs the batch keeps the 2-byte form."""
    n = 500
    rng = np.random.default_rng(3)
    shapes = np.array([0, 40, 97, 300, 1200])
    tok = rng.integers(-1, 12, n).astype(np.int32)
    node = shapes[rng.integers(0, len(shapes), n)].astype(np.int32)
    ref = np.stack([node.astype(np.int64), np.zeros(n, np.int64)], axis=1)
    nc = NodeCodes()
    ec = EventCodes(nc)
    b = EventBatch(tok, ref, np.zeros(1, np.uint8), node).narrowed(nc, ec)
    assert b.ev8 is not None and b.packed is b.ev8 and b.ev8.dtype == np.uint8
    pairs = ec.host.numpy().reshape(256, 2)
    assert np.array_equal(pairs[b.ev8, 0], tok) and np.array_equal(pairs[b.ev8, 1], node)
    assert b.wire(False, narrow8=True)[0] is b.ev8
    # the 2-byte halves are still there (stage() uses them)
    assert np.array_equal(nc.host.numpy()[b.node8], node)
    # codes are stable across batches; new pairs are appended
    n0 = ec.n
    b2 = EventBatch(tok[::-1].copy(), ref[::-1].copy(), np.zeros(1, np.uint8),
                    node[::-1].copy()).narrowed(nc, ec)
    assert ec.n == n0 and np.array_equal(b2.ev8, b.ev8[::-1])
    # more than 256 distinct pairs: the 2-byte form
    many_tok = np.repeat(np.arange(60, dtype=np.int32), 5)
    many_node = np.tile(shapes.astype(np.int32), 60)
    many = EventBatch(many_tok, np.stack([many_node.astype(np.int64), np.zeros(300, np.int64)], 1),
                      np.zeros(1, np.uint8), many_node).narrowed(nc, ec)
    assert many.ev8 is None and many.node8 is not None


def test_keys_layout():
    for n, cap, a16 in ((1, 8, True), (1000, 16000, True), (1000, 16000, False)):
        k_off, a_off, size = keys_layout(n, cap, a16)
        assert k_off >= 40 and a_off % 64 == 0 and a_off >= k_off + 2 * n
        assert size == a_off + cap * (2 if a16 else 4)
        k_off, a_off8, size8 = keys_layout(n, cap, a16, kb=1)  # u8 plan codes
        assert a_off8 % 64 == 0 and k_off + n <= a_off8 <= a_off
        assert size8 == a_off8 + cap * (2 if a16 else 4)


def _plan_rows(K, M, entries):
    """Raw live-plan rows; entries: per key (nm, na, n_map, pids, acts, utils,
    words) or None (an empty entry); unused slots hold garbage."""
    L = plan_layout_host(K, M)
    rows = np.random.default_rng(5).integers(0, 256, (len(entries), L["stride"]), dtype=np.uint8)
    for r, e in zip(rows, entries):
        nm, na, nmap, pids, acts, utils, words = e or (0, 0, 0, [], [], [], [])
        r[0], r[1], r[2], r[3] = nm, na, nmap, min(nmap, 1)
        r[L["off_pid"]:L["off_pid"] + 4 * nm] = np.array(pids, np.int32).view(np.uint8)
        r[L["off_comp"]:L["off_comp"] + nm] = 2
        r[L["off_act"]:L["off_act"] + 2 * na] = np.array(acts, np.uint16).view(np.uint8)
        r[L["off_util"]:L["off_util"] + 8 * na] = np.array(utils, np.float64).view(np.uint8)
        r[L["off_map"]:L["off_map"] + 8 * nmap] = np.array(words, np.uint64).view(np.uint8)
    return rows


def test_plan_codes_share_equal_entries():
    K, M = 4, 8
    a = (2, 1, 0, [3, 5], [0x301], [1.5], [])
    b = (1, 1, 1, [7], [0x300], [2.0], [9])
    rows = _plan_rows(K, M, [None, a, b, a, None, b, a])
    codes, rep = plan_codes(rows, K, M)
    assert codes[0] == 0xFF and codes[4] == 0xFF  # empty entries: no key needed
    assert codes[1] == codes[3] == codes[6] != codes[2] == codes[5]
    for key in (1, 2, 3, 5, 6):  # the representative has the same content
        r = rep[codes[key]]
        assert r in (1, 2) and (r == 1) == (codes[key] == codes[1])
    assert (rep[2:] == -1).all()
    # more than 255 distinct contents: no u8 form
    many = [(1, 0, 0, [i], [], [], []) for i in range(256)]
    assert plan_codes(_plan_rows(K, M, many), K, M) is None
    assert plan_codes(_plan_rows(K, M, many[:255]), K, M) is not None


def _word(bind, rank, bslot, age, unit):
    return np.uint64(bind | (rank << 32) | (bslot << 40) | (age << 48) | (unit << 56))


@pytest.mark.parametrize("key8", [False, True])
def test_expand_unit_references(key8):
    K, B, n = 4, 2, 3
    patterns = np.zeros(3, _native.PATTERN_DTYPE)
    # p0: mapped, 2 bindings, tool 0; p1: unmapped, tool 1; p2: mapped, 1 binding, tool 0
    patterns["target_tool"] = [0, 1, 0]
    patterns["n_bind"] = [2, 0, 1]
    patterns["flags"] = [1, 0, 1]
    patterns["p"] = [0.5, 0.4, 0.25]
    benefit = np.array([700.0, 300.0])
    n_keys = 2
    entries = (np.array([3, 0]), np.array([[0, 1, 2, -1], [-1] * 4], np.int32))
    n_pred = np.array([3, 0])
    n_act = np.array([2, 0])
    acts = np.zeros((n_keys, K), np.uint16)
    acts[0, 0] = 0 | (3 << 8) | (1 << 12)   # tool 0: rank 0, FULL level 3, partial level 1
    acts[0, 1] = 1 | (1 << 8) | (1 << 12)   # tool 1: rank 1 (tool only), level 1
    n_map = np.array([3, 0])
    n_units = np.array([2, 0])
    M = K * B
    words = np.zeros((n_keys, M), np.uint64)
    words[0, 0] = _word(10, 0, 0, 1, 0)  # p0 binding 0 -> unit 0
    words[0, 1] = _word(11, 0, 1, 1, 1)  # p0 binding 1 -> unit 1
    words[0, 2] = _word(12, 2, 0, 1, 0)  # p2 binding 0: the same resolution as unit 0
    plan = (n_pred, n_act, acts, n_map, n_units, words)
    keys = np.array([0, 0, 0xFFFF], np.uint16)
    # session 0: both units resolved (region 1); session 1: unit 0 unresolved
    arg = np.array([(1 << 11) | 5, (1 << 11) | 7, 0xFFFF, (1 << 11) | 9], np.uint16)
    fmt = (_native.PASTE_CF_ENTRY16 | _native.PASTE_CF_KEYS | _native.PASTE_CF_UNIQ
           | _native.PASTE_CF_ARG16)
    if key8:  # u8 plan codes: code 0 stands for key 0, 0xFF for no entry
        fmt |= _native.PASTE_CF_KEY8
        rep = np.full(256, -1, np.int64)
        rep[0] = 0
        plan = plan + (rep,)
        keys = np.array([0, 0, 0xFF], np.uint8)
    rec = CompactRecords(K, B, np.zeros(0, np.uint16), keys, arg, np.zeros(0, np.uint8), fmt,
                         entries, plan)
    r = rec.expand(patterns, benefit).session_major()
    assert r.n_pred.tolist() == [3, 3, 0] and r.n_act.tolist() == [2, 2, 0]
    pat = r.pred_pat.reshape(n, K)
    comp = r.pred_comp.reshape(n, K)
    parg = r.pred_arg.reshape(n, K, B)
    assert pat[0, :3].tolist() == [0, 1, 2] and pat[1, :3].tolist() == [0, 1, 2]
    assert comp[0, :3].tolist() == [C_FULL, C_TOOL_ONLY, C_FULL]
    assert comp[1, :3].tolist() == [C_PARTIAL, C_TOOL_ONLY, C_PARTIAL]
    ev0, ev1 = 1 * n + 0, 1 * n + 1
    assert parg[0, 0].tolist() == [(ev0 << 32) | 5, (ev0 << 32) | 7]
    assert parg[0, 2, 0] == (ev0 << 32) | 5  # the shared unit's reference
    assert parg[1, 0].tolist() == [-1, (ev1 << 32) | 9]
    assert parg[1, 2, 0] == -1
    lvl = r.act_level.reshape(n, K)
    apred = r.act_pred.reshape(n, K)
    util = r.act_util.reshape(n, K)
    assert apred[0, :2].tolist() == [0, 1] and lvl[0, :2].tolist() == [3, 1]
    assert lvl[1, :2].tolist() == [1, 1]  # PARTIAL rank 0: admitted at its partial level
    assert util[0, 0] == 0.5 * 700.0 and util[0, 1] == 0.4 * 300.0

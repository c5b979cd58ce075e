"""Native JSONL parse with payload tapes (csrc/ingest.cpp, paste_jsonl_parse)
== json.loads + _parse_record (events.py:165-184) + the host tape encoder
(tape.py): same valid rows in file order, first-appearance session ids,
sigs, the reference's error list, and byte-identical payload tapes (result
and args of every record, canonical scalar bytes: digits for ints and
integral floats, Python's repr for other floats)."""

import json
import random

import numpy as np
import pytest

from golden_io import golden
from paper_2603_18897_b200.ingest import parse_jsonl_raw
from paper_2603_18897_b200.tape import KeyTable, TapeArena

CASES = golden("ingest_golden.json")["cases"]


def _host_rows(text, bad_lines):
    recs = []
    for no, raw in enumerate(text.splitlines(), start=1):
        if raw.strip() and no not in bad_lines:
            recs.append(json.loads(raw))
    return recs


def _check(text, tr, bad_lines):
    recs = _host_rows(text, bad_lines)
    assert len(tr.columns["sig"]) == len(recs)
    arena = TapeArena(KeyTable(), keep_objects=False)
    for r in recs:
        arena.add(r.get("result"))
        arena.add(r.get("args"))
    hn, hd, hr = arena.arrays()
    nn, nd, nr = tr.tapes
    assert np.array_equal(hr.reshape(-1, 2), nr.reshape(-1, 2))
    if not recs:
        return
    assert len(hn) == len(nn)
    for f in ("type", "flags", "a", "b"):
        assert np.array_equal(hn[f], nn[f]), f
    hk = [arena.keys.names[k] if k >= 0 else None for k in hn["key"].tolist()]
    nk = [tr.keys.names[k] if k >= 0 else None for k in nn["key"].tolist()]
    assert hk == nk
    used = len(arena._data)
    assert len(nd) == max(used, 1) and bytes(hd[:used]) == bytes(nd[:used])
    sid = {}
    for r, s in zip(recs, tr.columns["session"].tolist()):
        assert sid.setdefault(str(r["session_id"]), len(sid)) == s
    tools = sorted({str(r["tool"]) for r in recs if r["kind"] == "tool_call"})
    assert tr.sigs.tools == tools
    for r, g in zip(recs, tr.columns["sig"].tolist()):
        exp = -1 if r["kind"] == "llm_step" else 2 * tools.index(str(r["tool"])) + (
            r["status"] == "success")
        assert g == exp


@pytest.mark.parametrize("i", range(len(CASES)))
def test_native_parse_matches_golden_and_host_tapes(i):
    case = CASES[i]
    tr = parse_jsonl_raw(case["text"])
    if tr is None:  # outside the exact subset: the host ingest decides
        return
    assert [[e.line, e.message] for e in tr.errors] == case["expected"]["errors"]
    _check(case["text"], tr, {line for line, _ in case["expected"]["errors"]})


SCALARS = [None, True, False, 0, 7, -123456789012345678901234567890, 1.5, -0.25, 1e-7, 1e22,
           1.0, -0.0, 2.5e-320, 123456.789, 0.1 + 0.2, 1 / 3, 5e-5, 1e-4, 9007199254740993.0,
           1e300, "", "x", "a b\tc", "ünï", "été", "q\"b\\s/", "\x00nul",
           "line\nbreak", "ſɐ˿"]


def _payload(rng, depth=0):
    r = rng.random()
    if depth > 3 or r < 0.45:
        return rng.choice(SCALARS)
    if r < 0.75:
        return {rng.choice(["k", "url", "é", "x y", "list"]) + str(i): _payload(rng, depth + 1)
                for i in range(rng.randint(0, 4))}
    return [_payload(rng, depth + 1) for _ in range(rng.randint(0, 4))]


@pytest.mark.parametrize("seed", range(6))
def test_native_payload_tapes_equal_host_encoder(seed):
    rng = random.Random(seed)
    lines = []
    for i in range(300):
        rec = {"session_id": f"s{rng.randint(0, 20)}", "seq": i,
               "kind": rng.choice(["tool_call"] * 4 + ["llm_step"]),
               "tool": rng.choice(["a", "b", "web_fetch"]),
               "status": rng.choice(["success", "fail"]), "t_start_ms": float(i),
               "t_end_ms": float(i) + 1}
        if rec["kind"] == "llm_step":
            rec["tool"] = ""
        if rng.random() < 0.8:
            rec["result"] = _payload(rng)
        if rng.random() < 0.8:
            rec["args"] = _payload(rng)
        items = list(rec.items())
        rng.shuffle(items)  # args before result, payloads before ids, ...
        lines.append(json.dumps(dict(items), ensure_ascii=rng.random() < 0.5))
    text = "\n".join(lines) + "\n"
    tr = parse_jsonl_raw(text)
    assert tr is not None
    _check(text, tr, set())


HEAD = ('{"session_id": "s", "seq": 0, "kind": "tool_call", "tool": "a", "status": "success", '
        '"t_start_ms": 1, "t_end_ms": 2, ')


@pytest.mark.parametrize("tail", [
    '"args": {"q": "e\\u0301"}}',      # a combining mark: NFC needs the Unicode database
    '"args": {"q": 1, "q": 2}}',       # duplicate key inside a payload
    '"result": "\\ud800"}',            # lone surrogate
    '"args": 1, "args": 2}',           # duplicate payload field
])
def test_outside_exact_subset_is_unsupported(tail):
    assert parse_jsonl_raw(HEAD + tail + "\n") is None

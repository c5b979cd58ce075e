"""Native columnar JSONL ingest (csrc/ingest.cpp) == the host ingest_trace
(events.py mirror of the reference's events.py:196-252) turned into the
columnar mining trace: same tool events, order, segment ids, sigs, error
lines and reordered-session count; inputs outside the native subset go to
the host path and give the same result."""

import io
import json
import random

import numpy as np
import pytest

from paper_2603_18897_b200 import ingest
from paper_2603_18897_b200.events import Event, EventKind, Session, Status, write_trace


def _trace(seed, n_sessions=300, interleave=True, extras=True, payloads=True):
    rng = random.Random(seed)
    tools = ["search", "web_fetch", "file_editor", "terminal", "grep", "zeta", "Alpha"]
    sessions = []
    for s in range(n_sessions):
        t = rng.uniform(0, 1e6)
        evs = []
        for q in range(rng.randint(1, 14)):
            kind = EventKind.LLM_STEP if rng.random() < 0.2 else EventKind.TOOL_CALL
            gap = rng.choice([10.0, 500.0, 250_000.0, 400_000.0, 299_999.5, 300_000.0])
            t += gap
            dur = rng.uniform(1, 2000)
            args = {"q": rng.randint(0, 9), "s": "é" * rng.randint(0, 2)} if rng.random() < 0.5 else None
            result = {"r": [1, 2.5, None, True]}
            if not payloads:
                args = result = None
            evs.append(Event(f"sess-{s}", q, kind, rng.choice(tools),
                             Status.FAIL if rng.random() < 0.1 else Status.SUCCESS,
                             args, result, t, t + dur))
        if rng.random() < 0.2 and len(evs) > 2:  # out-of-order timestamps
            i = rng.randrange(len(evs) - 1)
            a, b = evs[i], evs[i + 1]
            evs[i] = Event(a.session_id, a.seq, a.kind, a.tool_type, a.status, a.args, a.result,
                           b.t_start, b.t_end)
            evs[i + 1] = Event(b.session_id, b.seq, b.kind, b.tool_type, b.status, b.args,
                               b.result, a.t_start, a.t_end)
        sessions.append(Session(f"sess-{s}", tuple(evs)))
    buf = io.StringIO()
    write_trace(sessions, buf)
    lines = buf.getvalue().splitlines()
    if interleave:
        rng.shuffle(lines)
    if extras:
        for _ in range(10):  # records missing a field, blank lines
            rec = json.loads(rng.choice(lines))
            del rec[rng.choice(["seq", "tool", "t_end_ms", "kind"])]
            lines.insert(rng.randrange(len(lines)), json.dumps(rec))
            lines.insert(rng.randrange(len(lines)), "   ")
    return "\n".join(lines) + "\n"


def _assert_same(a, b):
    for k in ("session", "seq", "t_start", "t_end", "sig"):
        assert np.array_equal(a.columns[k], b.columns[k], equal_nan=k.startswith("t_")), k
    assert a.sigs.tools == b.sigs.tools
    assert a.n_segments == b.n_segments and a.reordered_sessions == b.reordered_sessions
    assert [(e.line, e.message) for e in a.errors] == [(e.line, e.message) for e in b.errors]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_native_ingest_equals_host_ingest(seed):
    text = _trace(seed)
    nat = ingest.ingest_columnar(text)
    assert nat.native and nat.n_events > 0 and len(nat.errors) == 10
    _assert_same(nat, ingest._host(text, 300_000.0))


@pytest.mark.parametrize("bad", [
    '{"session_id": "s\\"q", "seq": 0, "kind": "tool_call", "tool": "a", "status": "success", '
    '"t_start_ms": 1.0, "t_end_ms": 2.0}',                          # escaped id
    '{"session_id": 7, "seq": 0, "kind": "tool_call", "tool": "a", "status": "success", '
    '"t_start_ms": 1.0, "t_end_ms": 2.0}',                          # str(int) id
    '{"session_id": "s", "seq": 1.0, "kind": "tool_call", "tool": "a", "status": "success", '
    '"t_start_ms": 1.0, "t_end_ms": 2.0}',                          # int(float) seq
    '{"session_id": "s", "seq": 0, "kind": "tool_call", "tool": "a", "status": "success", '
    '"t_start_ms": NaN, "t_end_ms": 2.0}',                          # NaN sort key
    '[1, 2]',                                                       # not an object
])
def test_outside_native_subset_uses_host_semantics(bad):
    text = _trace(9, n_sessions=40, extras=False) + bad + "\n"
    res = ingest.ingest_columnar(text)
    assert not res.native
    _assert_same(res, ingest._host(text, 300_000.0))


def test_line_separators_python_would_split():
    text = _trace(4, n_sessions=20, extras=False).replace("\n", "\r\n")
    res = ingest.ingest_columnar(text)
    assert not res.native
    _assert_same(res, ingest._host(text, 300_000.0))


def test_post_init_rejections_are_ingest_errors():
    """Records Event.__post_init__ rejects (t_start > t_end; a tool_call with
    an empty tool) are tallied errors with the reference's messages, on the
    native path, not events (events.py:59-63)."""
    good = _trace(5, n_sessions=30, extras=False)
    bad = [
        '{"session_id": "s1", "seq": 4, "kind": "tool_call", "tool": "a", "status": "success", '
        '"t_start_ms": 5.0, "t_end_ms": 2.0}',
        '{"session_id": "s1", "seq": 5, "kind": "tool_call", "tool": "", "status": "fail", '
        '"t_start_ms": 1.0, "t_end_ms": 2.0}',
        '{"session_id": "s2", "seq": 6, "kind": "llm_step", "tool": "", "status": "success", '
        '"t_start_ms": 1.0, "t_end_ms": 2.0}',  # an LLM step may have an empty tool
        '{"session_id": "s3", "seq": 7, "kind": "llm_step", "tool": "", "status": "success", '
        '"t_start_ms": 9.0, "t_end_ms": 2.0}',
        '{"seq": 8, "tool": "", "status": "success", "t_start_ms": 9.0}',
    ]
    text = good + "\n".join(bad) + "\n"
    nat = ingest.ingest_columnar(text)
    assert nat.native
    host = ingest._host(text, 300_000.0)
    _assert_same(nat, host)
    msgs = [e.message for e in nat.errors]
    assert msgs == ["event seq=4: t_start > t_end", "event seq=5: tool_call with empty tool_type",
                    "event seq=7: t_start > t_end", "missing fields: session_id, kind, t_end_ms"]

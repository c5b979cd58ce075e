"""Ingestion pinned to the REFERENCE's ingest_trace (events.py:196-252):
tests/golden/ingest_golden.json holds JSONL texts and what the reference
returned for them (sessions with their events in order, #n segment ids, the
per-line error list, the reordered-session tally).  Checked here against
  * the host mirror's ingest_trace,
  * the native columnar ingest (csrc/ingest.cpp, or its host decision for
    input outside the native subset), projected to tool events,
and, in test_ingest_sort_gpu.py, the device K1 general path."""

import json

import numpy as np
import pytest

from golden_io import golden, session
from paper_2603_18897_b200 import ingest
from paper_2603_18897_b200.events import Status, event_to_record, ingest_trace

CASES = golden("ingest_golden.json")["cases"]


def _run_host(case):
    if case["threshold"] is None:
        return ingest_trace(case["text"])
    return ingest_trace(case["text"], case["threshold"])


def _same_record(a: dict, b: dict) -> bool:
    # json round trip of the reference's records: compare floats by value (NaN never
    # reaches a record: the reference raises on it only through the comparisons)
    return json.dumps(a, sort_keys=True) == json.dumps(b, sort_keys=True)


@pytest.mark.parametrize("i", range(len(CASES)))
def test_host_ingest_equals_reference(i):
    case = CASES[i]
    res = _run_host(case)
    exp = case["expected"]
    assert [s.session_id for s in res.sessions] == [s["id"] for s in exp["sessions"]]
    for s, es in zip(res.sessions, exp["sessions"]):
        got = [event_to_record(e) for e in s.events]
        assert len(got) == len(es["events"])
        assert all(_same_record(a, b) for a, b in zip(got, es["events"])), s.session_id
    assert [[e.line, e.message] for e in res.errors] == exp["errors"]
    assert res.reordered_sessions == exp["reordered"]


def expected_columns(case):
    """The reference's ingest result as the columnar mining trace: tool events
    of every segment in order, session = segment index, sig = 2 * (rank of
    the tool in sorted name order) + (status == success)."""
    sessions = [session(s) for s in case["expected"]["sessions"]]
    streams = [s.tool_events() for s in sessions]
    tools = sorted({e.tool_type for st in streams for e in st})
    tid = {t: i for i, t in enumerate(tools)}
    cols = {"session": [], "seq": [], "t_start": [], "t_end": [], "sig": []}
    for seg, st in enumerate(streams):
        for e in st:
            cols["session"].append(seg)
            cols["seq"].append(e.seq)
            cols["t_start"].append(e.t_start)
            cols["t_end"].append(e.t_end)
            cols["sig"].append(2 * tid[e.tool_type] + (e.status is Status.SUCCESS))
    dt = {"session": np.int32, "seq": np.int32, "t_start": np.float64, "t_end": np.float64,
          "sig": np.int32}
    return {k: np.asarray(v, dt[k]) for k, v in cols.items()}, tools, len(sessions)


@pytest.mark.parametrize("i", range(len(CASES)))
def test_native_columnar_ingest_equals_reference(i):
    case = CASES[i]
    thr = 300_000.0 if case["threshold"] is None else case["threshold"]
    got = ingest.ingest_columnar(case["text"], thr)
    cols, tools, n_seg = expected_columns(case)
    for k in cols:
        assert np.array_equal(got.columns[k], cols[k]), k
    assert got.sigs.tools == tools
    assert got.n_segments == n_seg
    assert got.reordered_sessions == case["expected"]["reordered"]
    assert [[e.line, e.message] for e in got.errors] == case["expected"]["errors"]


def test_golden_covers_the_edges():
    """The fixture exercises what the reference's ingest branches on."""
    ids = [s["id"] for c in CASES for s in c["expected"]["sessions"]]
    msgs = {m.split(":")[0] for c in CASES for _, m in c["expected"]["errors"]}
    assert any("#" in x for x in ids)
    assert sum(c["expected"]["reordered"] for c in CASES) >= 10
    assert any(m.startswith("event seq=") for m in msgs) and "missing fields" in msgs
    assert "record is not an object" in msgs
    assert any(c["threshold"] not in (None, 300_000.0) for c in CASES)

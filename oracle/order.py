"""CPU restatement of ingest_trace's grouping, stable sort, reorder tally and
gap split over a columnar trace in arrival order (TEST INFRASTRUCTURE ONLY:
imported by tests/ as the checker, never by the product package).

Follows /root/reference/pkg/src/spectool/events.py:
  * :221-225  group events by session in first-appearance order (here: by
              session id, the ids being first-appearance indices);
  * :230-233  ``sorted(events, key=lambda e: (e.t_start, e.seq))`` -- Python's
              sort is stable, so equal keys keep arrival order, and -0.0 ==
              0.0; a session is reordered when its seq list changed;
  * :234-240, :243-252  split where ``t_start - prev.t_end > threshold`` over
              every event (LLM steps included), then Session.tool_events
              (:66-72) keeps the tool calls of each segment.
Pinned against the reference's own ingest_trace output by
tests/test_order_oracle.py (tests/golden/ingest_golden.json).
"""

from __future__ import annotations

import numpy as np


def order_trace(session, seq, t_start, t_end, sig, n_sessions: int, threshold_ms: float):
    """Returns (columns dict of the tool events: session = global segment
    index, seq, t_start, t_end, sig), n_segments, reordered_sessions,
    order (arrival index of every event in sorted order)."""
    session = np.asarray(session, np.int64)
    seq = np.asarray(seq, np.int64)
    t_start = np.asarray(t_start, np.float64)
    t_end = np.asarray(t_end, np.float64)
    sig = np.asarray(sig, np.int64)
    n = len(session)
    arrival = np.arange(n)
    key_t = np.where(t_start == 0.0, 0.0, t_start)
    order = np.lexsort((arrival, seq, key_t, session))          # (session, t, seq, arrival)
    grouped = np.lexsort((arrival, session))                    # arrival order per session
    s_sorted = session[order]
    changed = seq[order] != seq[grouped]
    reordered = len(np.unique(s_sorted[changed]))
    first = np.ones(n, bool)
    first[1:] = s_sorted[1:] != s_sorted[:-1]
    gap = np.zeros(n, bool)
    gap[1:] = (t_start[order][1:] - t_end[order][:-1]) > threshold_ms
    new_seg = first | gap
    seg = np.cumsum(new_seg) - 1
    tool = sig[order] >= 0
    o = order[tool]
    cols = {"session": seg[tool].astype(np.int32), "seq": seq[o].astype(np.int32),
            "t_start": t_start[o], "t_end": t_end[o], "sig": sig[o].astype(np.int32)}
    return cols, int(new_seg.sum()), int(reordered), order.astype(np.int32)

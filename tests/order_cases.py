"""Raw arrival-order columns (the input of the K1 general path) from the
ingest goldens' JSONL texts, and a random interleaved trace generator."""

import json

import numpy as np


def raw_columns(case):
    """Every line the reference accepted (its error list names the rest), in
    file order: session = first-appearance index of str(session_id), sig =
    2 * (rank of the tool in sorted name order) + success, -1 for LLM steps
    (events.py:140-160 coercions)."""
    bad = {line for line, _ in case["expected"]["errors"]}
    recs = []
    for no, raw in enumerate(case["text"].splitlines(), start=1):
        if not raw.strip() or no in bad:
            continue
        recs.append(json.loads(raw))
    sid = {}
    tools = sorted({str(r["tool"]) for r in recs if r["kind"] == "tool_call"})
    tid = {t: i for i, t in enumerate(tools)}
    cols = {"session": [], "seq": [], "t_start": [], "t_end": [], "sig": []}
    for r in recs:
        cols["session"].append(sid.setdefault(str(r["session_id"]), len(sid)))
        cols["seq"].append(int(r["seq"]))
        cols["t_start"].append(float(r["t_start_ms"]))
        cols["t_end"].append(float(r["t_end_ms"]))
        cols["sig"].append(-1 if r["kind"] == "llm_step"
                           else 2 * tid[str(r["tool"])] + (r["status"] == "success"))
    dt = {"session": np.int32, "seq": np.int32, "t_start": np.float64, "t_end": np.float64,
          "sig": np.int32}
    return {k: np.asarray(v, dt[k]) for k, v in cols.items()}, len(sid)


def random_trace(n_sessions, seed, long_sessions=(), interleave=True):
    """Arrival-order columns: sessions of 1..40 events (plus the given long
    ones), timestamps mostly increasing with ties, swaps, duplicate (t, seq)
    pairs, -0.0, LLM steps and gaps around 300 s; ids in first-appearance
    order when interleaved."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 41, n_sessions)
    for i, L in enumerate(long_sessions):
        lens[(i * 7919) % n_sessions] = L
    n = int(lens.sum())
    sess = np.repeat(np.arange(n_sessions, dtype=np.int64), lens)
    pos = np.arange(n) - np.repeat(np.cumsum(lens) - lens, lens)
    step = rng.choice([0.0, 10.0, 500.0, 299_999.5, 300_000.0, 300_000.5, 4e5], n,
                      p=[.1, .5, .2, .05, .05, .05, .05])
    t = np.cumsum(step)
    t -= np.repeat(t[np.cumsum(lens) - lens], lens)
    t[rng.random(n) < 0.02] = -0.0
    seq = pos.copy()
    dup = rng.random(n) < 0.03
    seq[dup] = np.maximum(seq[dup] - 1, 0)
    # local disorder: swap some neighbours' timestamps inside a session
    sw = np.flatnonzero((rng.random(n - 1) < 0.05) & (sess[1:] == sess[:-1]))
    t[sw], t[sw + 1] = t[sw + 1].copy(), t[sw].copy()
    dur = rng.choice([0.0, 1.0, 250.0], n)
    sig = rng.integers(0, 24, n)
    sig[rng.random(n) < 0.15] = -1
    arrival = np.arange(n)
    if interleave:
        arrival = np.argsort(rng.random(n) + sess * 0.002, kind="stable")
        sess_arr = sess[arrival]
        first = {}
        for s in sess_arr:
            first.setdefault(int(s), len(first))
        remap = np.array([first[i] for i in range(n_sessions)], np.int64)
        sess = remap[sess]
    cols = {"session": sess[arrival].astype(np.int32), "seq": seq[arrival].astype(np.int32),
            "t_start": t[arrival], "t_end": (t + dur)[arrival], "sig": sig[arrival].astype(np.int32)}
    return cols
